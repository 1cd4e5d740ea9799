python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --workload cone4d2048 --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2n_c.json 2>gpurun_out/r2n.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cone or full_size or deterministic" > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2n_pytest.log
