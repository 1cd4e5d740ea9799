timeout 600 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_sl.so libdinr.so libdinr_var_sl.so libdinr.so libdinr_var_sl.so > gpurun_out/r4b_variants.txt 2>&1
