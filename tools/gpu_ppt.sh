# chunk size experiment (pixels per thread cap) under the tiled CTA order, full c4
for p in 32 16 64 8 32; do
  PBA_PPT_MAX=$p timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ppt_$p.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ppt_$p.log').read().strip().splitlines()[-1]);print('ppt$p step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
done
