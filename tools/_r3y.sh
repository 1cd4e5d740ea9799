python -c "import __graft_entry__ as g; g.build()"
if ! timeout 180 python tools/variant_time.py cone4d2048 libdinr.so > gpurun_out/r3y_quick.txt 2>&1; then echo "quick check failed/hung" >> gpurun_out/r3y_quick.txt; exit 3; fi
timeout 700 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r3y_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3y_pytest.log
timeout 400 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_fq0.so libdinr.so libdinr_var_fq0.so > gpurun_out/r3y_variants.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3y_bench.jsonl 2>>gpurun_out/r3y_bench.err
