# c1 (the reference's own small case): chunk-size sweep and the launch list of the timed steps
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e-api > gpurun_out/c1_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/c1_$tag.log').read().strip().splitlines()[-1]);print('$tag','step ms',round(d['ms_per_step'],4),'lin ms',round(d['roofline']['linearize_ms'],4))"
}
for i in 1 2; do
  run def$i
  for u in 3 5; do run u${u}_$i PBA_CHUNK_UNITS=$u; done
done
PBA_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/c1_ncu.log 2>&1; echo "ncu rc=$?"
