python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_z0.so libdinr_var_hs4.so libdinr.so libdinr_var_z0.so libdinr_var_hs4.so > gpurun_out/r3q_variants.txt 2>&1
timeout 300 python tools/phases3.py > gpurun_out/r3q_phases.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r3q_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3q_pytest.log
