set -x
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 900 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1]);print('step ms',d['ms_per_step'],'lin ms',d['roofline']['linearize_ms'],'solve ms',d['roofline']['solve_ms'],'frac',d['roofline']['frac'], 'e2e', d['e2e']['ms_per_step'])"
