# K1 chunk size sweep (PBA_CHUNK_UNITS x 256 pixels per CTA) on c4/200
for u in ${UNITS:-32 16 48 64 32}; do
  PBA_CHUNK_UNITS=$u timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/chunk_$u.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/chunk_$u.log').read().strip().splitlines()[-1]);print('units $u','step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
