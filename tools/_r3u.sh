python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r3u_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3u_pytest.log
timeout 900 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_s0.so libdinr_var_f0.so libdinr_var_b0.so libdinr.so libdinr_var_s0.so > gpurun_out/r3u_variants.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3u_bench.jsonl 2>>gpurun_out/r3u_bench.err
