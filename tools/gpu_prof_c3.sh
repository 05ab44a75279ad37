# ncu --set full of K1 on the pinhole c3 workload (100 frames), after a clean run
CMD="python bench.py --config c3 --frames 100 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-api"
timeout 600 $CMD > gpurun_out/c3_small.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/c3_small.log | cut -c1-300
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:linearize_kernel -s 3 -c 1 -o gpurun_out/prof_linearize_c3 -f $CMD > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
