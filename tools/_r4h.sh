for i in 1 2 3; do
  timeout 150 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_wl.so libdinr_var_de.so >> gpurun_out/r4h_variants.txt 2>&1
done
