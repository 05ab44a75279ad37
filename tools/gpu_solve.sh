set -x
timeout 300 python tools/solve_bench.py --dense > gpurun_out/solve_bench.log 2>&1; echo "rc=$?"; cat gpurun_out/solve_bench.log
timeout 300 python tools/solve_bench.py --reps 1 > gpurun_out/solve_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches.csv python tools/solve_bench.py --reps 1 > gpurun_out/ncu_solve.log 2>&1; echo "ncu rc=$?"
