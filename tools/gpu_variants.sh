run() { # tag env...
  tag=$1; shift
  env "$@" timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_$tag.log 2>&1; echo "$tag rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/var_$tag.log').read().strip().splitlines()[-1]);print('$tag','step ms',d['ms_per_step'],'lin ms',d['roofline']['linearize_ms'],'frac',d['roofline']['frac'])"
}
for v in ${VARIANTS:-4 15 16 4}; do run v$v PBA_LIN_VARIANT=$v; done
