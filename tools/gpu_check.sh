set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 900 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.log 2>&1; echo "bench c1 rc=$?"
tail -5 gpurun_out/bench_c1.log
timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 > gpurun_out/bench_c4_200.log 2>&1; echo "bench c4-200 rc=$?"
tail -5 gpurun_out/bench_c4_200.log
