# chunk-order tile size sweep (PBA_CHUNK_BLOCK) for the current K1: c4/200 and c3/100
run() { # tag config frames env...
  tag=$1; cfg=$2; fr=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --frames $fr --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/blk_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/blk_$tag.log').read().strip().splitlines()[-1]);print('$tag','step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
}
run c4_def c4 200
for b in 8 12 24 32; do run c4_b$b c4 200 PBA_CHUNK_BLOCK=$b; done
run c3_def c3 100
for b in 16 24 48 64; do run c3_b$b c3 100 PBA_CHUNK_BLOCK=$b; done
