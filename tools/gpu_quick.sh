set -x
python -c "from oracle import oracle; oracle.build(force=True)"
timeout 900 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python tools/probe_costonly.py 200
timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1]);print('step ms',d['ms_per_step'],'lin ms',d['roofline']['linearize_ms'],'frac',d['roofline']['frac'])"
