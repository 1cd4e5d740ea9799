timeout 200 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r4k_bench.json 2>gpurun_out/r4k.err
timeout 200 python bench.py --workload fan512 --steps 10 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r4k_bench_fan.json 2>>gpurun_out/r4k.err
