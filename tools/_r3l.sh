python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/r3l_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3l_pytest.log
for i in 1 2; do
  timeout 400 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3l_bench.jsonl 2>>gpurun_out/r3l_bench.err
  DINR_F3_BULK_H=1 timeout 400 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3l_bench_bulk.jsonl 2>>gpurun_out/r3l_bench.err
done
for w in cone512 cone4d512; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3l_bench_other.jsonl 2>>gpurun_out/r3l_bench.err
done
