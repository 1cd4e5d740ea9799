python -c "import __graft_entry__ as g; g.build()"
for w in cone4d2048 cone512 cone4d512 fan512 parallel64; do
  timeout 200 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r4n_bench_$w.json 2>>gpurun_out/r4n.err
done
timeout 200 python bench.py --full-step --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r4n_bench_full.json 2>>gpurun_out/r4n.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r4n_reference.json 2>>gpurun_out/r4n.err
