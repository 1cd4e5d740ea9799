python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_noz.so libdinr_var_noh.so libdinr_var_nozh.so libdinr.so > gpurun_out/r3n_variants.txt 2>&1
DINR_F3_PACKED=1 timeout 300 python tools/variant_time.py cone4d2048 libdinr.so >> gpurun_out/r3n_variants.txt 2>&1
timeout 300 python tools/phases3.py > gpurun_out/r3n_phases.txt 2>&1
DINR_F3_PACKED=1 timeout 300 python tools/phases3.py > gpurun_out/r3n_phases_pk.txt 2>&1
