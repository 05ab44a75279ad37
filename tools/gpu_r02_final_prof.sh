# final round-2 captures: launch list of the default bench command (full c4) and one ncu --set full of K1 on it
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e-api"
timeout 900 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launches_c4.log 2>&1; echo "ncu launches rc=$?"
CMD3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-api"
timeout 900 $CMD3 > gpurun_out/plain_full1.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:linearize_kernel -s 4 -c 1 -o gpurun_out/prof_lin_c4full -f $CMD3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
