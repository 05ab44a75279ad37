# GPU suite + smoke + default bench (with cpu_baseline and e2e_api) + reference arm
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 1500 python -m pytest tests -m gpu -q --tb=short --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_reference.log 2>&1; echo "bench ref rc=$?"
tail -c 1500 gpurun_out/bench_reference.log
