# round-2 opening run on one B200: GPU suite, smoke, default bench, ncu launch list of c4/200
set -x
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log
CMD2="python bench.py --config c4 --frames 200 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD2 > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
