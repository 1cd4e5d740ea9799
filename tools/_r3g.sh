python -c "import __graft_entry__ as g; g.build()"
timeout 600 bash -c 'DINR_ZALL=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "cone or full"' > gpurun_out/r3g_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3g_pytest.log
for i in 1 2; do
DINR_ZALL=1 timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3g_zall_$i.json 2>>gpurun_out/r3g.err
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3g_def_$i.json 2>>gpurun_out/r3g.err
done
