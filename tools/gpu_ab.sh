# quick A/B after a K1 change: c4/200 x3 and c3/100 x2 (no tests)
for i in 1 2 3; do
  timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c4_$i.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_c4_$i.log').read().strip().splitlines()[-1]);print('c4/200 run $i step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
for i in 1 2; do
  timeout 900 python bench.py --config c3 --frames 100 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c3_$i.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_c3_$i.log').read().strip().splitlines()[-1]);print('c3/100 run $i step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
