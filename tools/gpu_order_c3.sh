# tile block-size sweep on the full c3 (pinhole 640x480) workload
for b in 16 24 32 48 16; do
  PBA_CHUNK_BLOCK=$b timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/oc3_b$b.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/oc3_b$b.log').read().strip().splitlines()[-1]);print('c3 b$b step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
