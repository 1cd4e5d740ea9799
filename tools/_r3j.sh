python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3j_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3j_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3j_smoke.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r3j_bench.json 2>gpurun_out/r3j_bench.err
timeout 400 python bench.py --workload parallel64 --steps 20 --warmup 5 > gpurun_out/r3j_bench_p64.json 2>>gpurun_out/r3j_bench.err
