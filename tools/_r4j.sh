for b in 48 768 2048 8192; do timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r4j_batch_$b.json 2>>gpurun_out/r4j.err; done
timeout 300 python bench.py --workload cone512 --batch 6144 --strong --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r4j_strong6144.json 2>>gpurun_out/r4j.err
