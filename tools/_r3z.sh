python -c "import __graft_entry__ as g; g.build()"
if ! timeout 180 python tools/variant_time.py cone4d2048 libdinr.so > gpurun_out/r3z_quick.txt 2>&1; then echo "quick check failed/hung" >> gpurun_out/r3z_quick.txt; exit 3; fi
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r3z_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3z_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3z_smoke.log 2>&1
for w in cone4d2048 cone512 cone4d512 fan512 parallel64; do
  timeout 200 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r3z_bench_$w.json 2>>gpurun_out/r3z_bench.err
done
timeout 200 python bench.py --full-step --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3z_bench_full.json 2>>gpurun_out/r3z_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r3z_reference.json 2>>gpurun_out/r3z_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3z_launches.csv python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r3z_ncu_launch.log 2>&1
B="python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_fwd3 -c 1 -o gpurun_out/r3z_fwd3 $B > gpurun_out/r3z_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_bwd3 -c 1 -o gpurun_out/r3z_bwd3 $B > gpurun_out/r3z_ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_dw -c 1 -o gpurun_out/r3z_dw $B > gpurun_out/r3z_ncu3.log 2>&1
timeout 700 python tests/_fuzz_parity.py 100 8675309 > gpurun_out/r3z_fuzz100.jsonl 2>&1; echo "rc $?" >> gpurun_out/r3z_fuzz100.jsonl
