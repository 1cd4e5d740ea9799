python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_paths.py -m gpu -q > gpurun_out/r3m_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3m_pytest.log
for i in 1 2; do
  timeout 400 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3m_bench.jsonl 2>>gpurun_out/r3m_bench.err
  DINR_F3_PACKED=1 timeout 400 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3m_bench_pk.jsonl 2>>gpurun_out/r3m_bench.err
done
DINR_F3_PACKED=1 timeout 1200 python tests/_fuzz_parity.py 120 4242 > gpurun_out/r3m_fuzz_pk.jsonl 2>&1; echo "rc $?" >> gpurun_out/r3m_fuzz_pk.jsonl
