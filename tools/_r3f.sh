python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py -q > gpurun_out/r3f_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3f_pytest.log
for b in 48 768 2048 8192; do timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3f_batch_$b.json 2>>gpurun_out/r3f.err; done
timeout 300 python bench.py --workload cone512 --batch 6144 --strong --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3f_strong6144.json 2>>gpurun_out/r3f.err
