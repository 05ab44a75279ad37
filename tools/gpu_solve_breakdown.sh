# per-kernel warm-cache durations of the banded dim-5994 solve (ncu, cache control off)
timeout 300 python tools/solve_bench.py --dim 5994 --band 126 --reps 3 > gpurun_out/sb_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/sb_plain.log
timeout 900 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/solve_launches.csv python tools/solve_bench.py --dim 5994 --band 126 --reps 3 > gpurun_out/sb_ncu.log 2>&1; echo "ncu rc=$?"
