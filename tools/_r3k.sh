python -c "import __graft_entry__ as g; g.build()"
for w in cone4d2048 cone512 cone4d512 fan512 parallel64; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r3k_bench_$w.json 2>>gpurun_out/r3k_bench.err
done
timeout 400 python bench.py --full-step --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3k_bench_full.json 2>>gpurun_out/r3k_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r3k_reference.json 2>>gpurun_out/r3k_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3k_launches.csv python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r3k_ncu_launch.log 2>&1
B="python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_fwd3 -c 1 -o gpurun_out/r3k_fwd3 $B > gpurun_out/r3k_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_bwd3 -c 1 -o gpurun_out/r3k_bwd3 $B > gpurun_out/r3k_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_dw -c 1 -o gpurun_out/r3k_dw $B > gpurun_out/r3k_ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r3k_fan512 $B --workload fan512 > gpurun_out/r3k_ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r3k_p64 $B --workload parallel64 > gpurun_out/r3k_ncu5.log 2>&1
