python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python tests/_fuzz_parity.py 300 271828 > gpurun_out/r4c_fuzz300.jsonl 2>&1; echo "rc $?" >> gpurun_out/r4c_fuzz300.jsonl
DINR_FUZZ_DEEP=1 timeout 900 python tests/_fuzz_parity.py 150 314159 > gpurun_out/r4c_fuzz_deep.jsonl 2>&1; echo "rc $?" >> gpurun_out/r4c_fuzz_deep.jsonl
DINR_FUZZ_PHANTOM_Y=1 timeout 900 python tests/_fuzz_parity.py 150 161803 > gpurun_out/r4c_fuzz_phantom.jsonl 2>&1; echo "rc $?" >> gpurun_out/r4c_fuzz_phantom.jsonl
