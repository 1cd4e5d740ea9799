python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3d_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3d_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3d_smoke.log 2>&1
for w in cone4d2048 cone512 cone4d512 fan512 parallel64; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r3d_bench_$w.json 2>>gpurun_out/r3d_bench.err
done
timeout 400 python bench.py --full-step --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3d_bench_full.json 2>>gpurun_out/r3d_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r3d_reference.json 2>>gpurun_out/r3d_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3d_launches.csv python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r3d_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_fwd3 -c 1 -o gpurun_out/r3d_fwd3 python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r3d_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_mlp -c 1 -o gpurun_out/r3d_k3 python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r3d_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_dw -c 1 -o gpurun_out/r3d_k5 python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r3d_ncu3.log 2>&1
