python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_pipeline_depth.py tests/test_gpu_paths.py -m gpu -q > gpurun_out/r4a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4a_pytest.log
