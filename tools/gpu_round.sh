# full round on one B200: GPU tests, default bench, reference arm, ncu launch list + one full capture
set -x
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 900 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log
timeout 1200 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "bench ref rc=$?"
tail -1 gpurun_out/bench_reference.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_default.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
CMD2="python bench.py --config c4 --frames 200 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:linearize_kernel -s 3 -c 1 -o gpurun_out/prof_linearize -f $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
