python -c "import __graft_entry__ as g; g.build()"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r4l_launches.csv python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r4l_ncu_launch.log 2>&1
B="python bench.py --steps 2 --warmup 3 --cpu-baseline-seconds 0"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_fwd3 -c 1 -o gpurun_out/r4l_fwd3 $B > gpurun_out/r4l_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_bwd3 -c 1 -o gpurun_out/r4l_bwd3 $B > gpurun_out/r4l_ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_dw -c 1 -o gpurun_out/r4l_dw $B > gpurun_out/r4l_ncu3.log 2>&1
timeout 300 python -m pytest tests/test_bench_contract.py -m gpu -q > gpurun_out/r4l_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4l_pytest.log
