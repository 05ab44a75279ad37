timeout 300 python tools/solve_bench.py --reps 1 > gpurun_out/solve_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:potrf -s 20 -c 1 -o gpurun_out/prof_potrf_la -f python tools/solve_bench.py --reps 1 > gpurun_out/ncu_potrf.log 2>&1; echo "ncu rc=$?"
