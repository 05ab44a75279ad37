timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
for c in c3 c5; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]);print('$c step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3),'solve',d['roofline']['solve_ms'],d['value']/1e9)"
done
