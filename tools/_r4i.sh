python -c "import __graft_entry__ as g; g.build()"
if ! timeout 180 python tools/variant_time.py cone4d2048 libdinr.so > gpurun_out/r4i_quick.txt 2>&1; then echo "quick check failed/hung" >> gpurun_out/r4i_quick.txt; exit 3; fi
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r4i_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4i_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4i_smoke.log 2>&1
for w in cone4d2048 cone4d512 cone512; do
  timeout 200 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r4i_bench_$w.json 2>>gpurun_out/r4i_bench.err
done
timeout 200 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r4i_bench_cone4d2048_b.json 2>>gpurun_out/r4i_bench.err
