# ncu --set full with source counters of K1 on c4/200 (one launch after warm-up), lean default
CMD2="python bench.py --config c4 --frames 200 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-api"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:linearize_kernel -s 3 -c 1 -o gpurun_out/prof_lin_small -f $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
