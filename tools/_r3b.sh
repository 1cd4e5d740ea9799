python -c "import __graft_entry__ as g; g.build()"
git -C . stash list > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_paths.py -q -x -k "cone or full or path" > gpurun_out/r3b_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3b_pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3b_c_$i.json 2>>gpurun_out/r3b.err; done
