# quick A/B on c4/200 (run after a K1 change): GPU suite, then three bench repetitions
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
for i in 1 2 3; do
  timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/quick_$i.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/quick_$i.log').read().strip().splitlines()[-1]);print('run $i step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
