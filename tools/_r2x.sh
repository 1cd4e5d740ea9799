python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_paths.py -q -x > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2x_pytest.log
for i in 1 2; do timeout 300 python bench.py --workload cone4d2048 --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2x_c_$i.json 2>>gpurun_out/r2x.err; done
timeout 300 python bench.py --workload cone512 --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2x_c512.json 2>>gpurun_out/r2x.err
