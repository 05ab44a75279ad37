# A/B of K1 variants on the full bench configs (one process per run)
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/ab_$tag.log 2>&1; echo "$tag rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1]);print('$tag','step ms',round(d['ms_per_step'],2),'lin ms',round(d['roofline']['linearize_ms'],2))"
}
for c in ${CONFIGS:-c4}; do
  for v in ${VARIANTS:-4 6 4 6}; do run ${c}_v$v $c PBA_LIN_VARIANT=$v; done
done
