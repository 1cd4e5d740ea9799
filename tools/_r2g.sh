python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python tests/_fuzz_parity.py 400 5151 > gpurun_out/r2g_fuzz400.jsonl 2>&1
timeout 900 python tests/_fuzz_parity.py 200 8080 > gpurun_out/r2g_fuzz200.jsonl 2>&1
DINR_FUZZ_PHANTOM_Y=1 timeout 900 python tests/_fuzz_parity.py 200 8080 > gpurun_out/r2g_fuzz200_phantom.jsonl 2>&1
python tools/variant_time.py fan512 libdinr.so > gpurun_out/r2g_vt_fan.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_fwd2 -c 1 -o gpurun_out/r2g_fwd2 python bench.py --workload cone4d2048 --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r2g_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_mlp -c 1 -o gpurun_out/r2g_bwd python bench.py --workload cone4d2048 --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r2g_ncu2.log 2>&1
