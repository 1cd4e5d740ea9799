for i in 1 2; do
for v in libdinr.so libdinr_var_v1.so libdinr_var_v2.so; do
  DINR_FWD4=1 timeout 120 python tools/variant_time.py cone4d2048 $v >> gpurun_out/r4e_variants.txt 2>&1
done
done
