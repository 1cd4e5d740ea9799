python -c "import __graft_entry__ as g; g.build()"
python tools/variant_time.py fan512 libdinr.so libdinr_var_pd.so libdinr_var_ps.so libdinr_var_pp.so > gpurun_out/r2f_vt_fan.txt 2>&1
for v in libdinr.so libdinr_var_pd.so libdinr_var_ps.so; do DINR_LIB=$v DINR_FUZZ_ONLY=100,271 python tests/_fuzz_parity.py 400 4242 > gpurun_out/r2f_fz_$v.jsonl 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2f_pytest.log 2>&1; echo pytest rc $? >> gpurun_out/r2f_pytest.log
for w in cone4d2048 cone512; do python bench.py --workload $w --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2f_$w.json 2>gpurun_out/r2f_$w.err; DINR_NO_BWD2=1 python bench.py --workload $w --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2f_${w}_nobwd2.json 2>>gpurun_out/r2f_$w.err; done
