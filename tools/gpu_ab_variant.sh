# A/B of K1 kernel variants (PBA_LIN_VARIANT) on one config, alternating, one
# process per run; then the parity suite under the candidate variant.
#   VARIANTS="6 7" CFG=c4 FRAMES=200 bash tools/gpu_ab_variant.sh
run() { # tag variant
  PBA_LIN_VARIANT=$2 timeout 900 python bench.py --config ${CFG:-c4} ${FRAMES:+--frames $FRAMES} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/abv_$1.log 2>&1; echo "$1 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/abv_$1.log').read().strip().splitlines()[-1]);print('$1','step ms',round(d['ms_per_step'],3),'lin ms',round(d['roofline']['linearize_ms'],3))"
}
V=(${VARIANTS:-6 7})
for i in 1 2; do for v in "${V[@]}"; do run v${v}_$i $v; done; done
if [ -n "${PARITY-1}" ]; then
  PBA_LIN_VARIANT=${V[-1]} timeout 1200 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_configs.py -k "not c2_full and not c3" 2>&1 | tail -5
fi
