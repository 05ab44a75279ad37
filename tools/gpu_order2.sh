# chunk order: destination-interleaved vs (source block x destination block) tiles
run() { # tag cfg frames env...
  tag=$1; c=$2; f=$3; shift 3
  env "$@" timeout 900 python bench.py --config $c --frames $f --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/order2_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/order2_$tag.log').read().strip().splitlines()[-1]);print('$tag step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
}
for c in "c3 100" "c4 200"; do
  set -- $c
  run $1_dst $1 $2 PBA_CHUNK_ORDER=dst
  run $1_blk2 $1 $2 PBA_CHUNK_ORDER=blk PBA_CHUNK_BLOCK=2
  run $1_blk4 $1 $2 PBA_CHUNK_ORDER=blk PBA_CHUNK_BLOCK=4
  run $1_blk8 $1 $2 PBA_CHUNK_ORDER=blk PBA_CHUNK_BLOCK=8
  run $1_dst2 $1 $2 PBA_CHUNK_ORDER=dst
done
