set -x
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 900 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_200.log 2>&1; echo "bench c4-200 rc=$?"
tail -3 gpurun_out/bench_c4_200.log
