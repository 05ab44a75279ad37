# GPU suite + default bench (c4) + c3/c5 lines after a change to K1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
for c in c3 c5; do timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
for f in bench_default bench_c3 bench_c5; do python -c "import json;d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]);print('$f step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3),'e2e',d['e2e']['ms_per_step'] if d.get('e2e') else None,'frac',d['roofline']['frac'],d['value']/1e9)"; done
