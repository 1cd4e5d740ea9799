python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3v_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3v_pytest.log
timeout 900 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_s1.so libdinr.so libdinr_var_s1.so > gpurun_out/r3v_variants.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 >> gpurun_out/r3v_bench.jsonl 2>>gpurun_out/r3v_bench.err
