set -x
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_pyramid.py -m gpu -q --tb=short > gpurun_out/pytest_pyr.log 2>&1; echo "pytest pyr rc=$?"
tail -30 gpurun_out/pytest_pyr.log
timeout 300 python tools/pyramid_bench.py --frames 64 > gpurun_out/pyr_bench.log 2>&1; echo "pyr bench rc=$?"; tail -3 gpurun_out/pyr_bench.log
timeout 900 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/var.log
