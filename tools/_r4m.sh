python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_bench_contract.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r4m_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4m_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4m_smoke.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r4m_reference.json 2>gpurun_out/r4m.err
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r4m_bench.json 2>>gpurun_out/r4m.err
