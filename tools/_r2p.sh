python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --workload cone4d2048 --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2p_c.json 2>gpurun_out/r2p.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2p_pytest.log
timeout 300 python bench.py --workload cone512 --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2p_c512.json 2>>gpurun_out/r2p.err
