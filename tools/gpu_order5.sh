# chunk order: rectangular (source x destination) tiles on the full c4 workload
run() { tag=$1; shift
  env "$@" timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/order5_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/order5_$tag.log').read().strip().splitlines()[-1]);print('$tag step',round(d['ms_per_step'],3),'lin',round(d['roofline']['linearize_ms'],3))"
}
run s16d16 PBA_CHUNK_BLOCK=16
run s16d32 PBA_CHUNK_BLOCK=16 PBA_CHUNK_BLOCK_DST=32
run s32d16 PBA_CHUNK_BLOCK=32 PBA_CHUNK_BLOCK_DST=16
run s8d16 PBA_CHUNK_BLOCK=8 PBA_CHUNK_BLOCK_DST=16
run s16d8 PBA_CHUNK_BLOCK=16 PBA_CHUNK_BLOCK_DST=8
run s16d1000 PBA_CHUNK_BLOCK=16 PBA_CHUNK_BLOCK_DST=1000
run s16d16b PBA_CHUNK_BLOCK=16
