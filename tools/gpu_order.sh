# K1 launch order of chunks: edge order vs destination- / source-interleaved
for cfg in "c3 100" "c4 200"; do
  set -- $cfg
  for o in pair dst src pair; do
    PBA_CHUNK_ORDER=$o timeout 900 python bench.py --config $1 --frames $2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/order_$1_$o.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/order_$1_$o.log').read().strip().splitlines()[-1]);print('$1 $o step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3),'cost0',d['config']['initial_cost'])"
  done
done
