# every bench line with the current code: default (c4, with cpu_baseline), c1, c2, c3, c5
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "c4 rc=$?"
for c in c1 c2 c3 c5; do timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
for f in bench_default bench_c1 bench_c2 bench_c3 bench_c5; do python -c "import json;d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]);print('$f step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3),'solve',d['roofline']['solve_ms'],'G/s',round(d['value']/1e9,2),'traffic',d['roofline']['traffic'])"; done
