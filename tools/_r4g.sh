for i in 1 2 3; do
  timeout 120 python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_ef.so >> gpurun_out/r4g_variants.txt 2>&1
done
