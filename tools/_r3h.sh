python -c "import __graft_entry__ as g; g.build()"
python -m paper_2404_19075_b200.build --variant sleep -DDINR_SLEEP_WAITS > /dev/null
python tools/variant_time.py cone4d2048 libdinr.so libdinr_var_sleep.so libdinr.so libdinr_var_sleep.so libdinr.so libdinr_var_sleep.so > gpurun_out/r3h_vt.txt 2>&1
python tools/variant_time.py cone512 libdinr.so libdinr_var_sleep.so libdinr.so libdinr_var_sleep.so > gpurun_out/r3h_vt512.txt 2>&1
