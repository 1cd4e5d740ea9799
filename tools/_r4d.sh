python -c "import __graft_entry__ as g; g.build()"
if ! DINR_FWD4=1 timeout 180 python tools/variant_time.py cone4d2048 libdinr.so > gpurun_out/r4d_quick.txt 2>&1; then echo "quick check failed/hung" >> gpurun_out/r4d_quick.txt; exit 3; fi
timeout 600 python -m pytest tests/test_gpu_paths.py -m gpu -q -k "FWD4" > gpurun_out/r4d_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4d_pytest.log
for i in 1 2; do
  timeout 120 python tools/variant_time.py cone4d2048 libdinr.so >> gpurun_out/r4d_variants.txt 2>&1
  DINR_FWD4=1 timeout 120 python tools/variant_time.py cone4d2048 libdinr.so >> gpurun_out/r4d_variants.txt 2>&1
done
DINR_FWD4=1 timeout 200 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r4d_bench.jsonl 2>>gpurun_out/r4d_bench.err
