# chunk order block-size sweep on the full c4 bench workload
for b in 16 8 12 20 24 16; do
  PBA_CHUNK_BLOCK=$b timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/order4_b$b.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/order4_b$b.log').read().strip().splitlines()[-1]);print('b$b step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
