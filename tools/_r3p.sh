for v in libdinr_phases.so libdinr_phases_dinr_dbg_no_hstore.so libdinr_phases_dinr_dbg_no_zstore.so libdinr_phases_dinr_dbg_no_hstore_dinr_dbg_no_zstore.so; do
  echo "== $v" >> gpurun_out/r3p_phases.txt
  DINR_PHASES_LIB=$v timeout 300 python tools/phases3.py 2>&1 | tail -1 >> gpurun_out/r3p_phases.txt
done
