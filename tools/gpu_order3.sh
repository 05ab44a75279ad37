# chunk order: block size sweep for the (source block x destination block) tiles
run() { # tag cfg frames env...
  tag=$1; c=$2; f=$3; shift 3
  env "$@" timeout 900 python bench.py --config $c --frames $f --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/order3_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/order3_$tag.log').read().strip().splitlines()[-1]);print('$tag step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
}
run c4_dst c4 200 PBA_CHUNK_ORDER=dst
for b in 8 12 16 24 32 64; do run c4_blk$b c4 200 PBA_CHUNK_ORDER=blk PBA_CHUNK_BLOCK=$b; done
run c4_pair c4 200 PBA_CHUNK_ORDER=pair
run c3_dst c3 100 PBA_CHUNK_ORDER=dst
for b in 16 32; do run c3_blk$b c3 100 PBA_CHUNK_ORDER=blk PBA_CHUNK_BLOCK=$b; done
