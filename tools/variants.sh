set -x
for m in 2 3 4 5; do
PBA_LIN_VARIANT=$m timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_$m.log 2>&1; echo "variant $m rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/var_$m.log').read().strip().splitlines()[-1]);print('variant',$m,'step ms',d['ms_per_step'],'lin ms',d['roofline']['linearize_ms'],'frac',d['roofline']['frac'], 'e2e', d['e2e']['ms_per_step'])"
done
CMD="python bench.py --config c4 --frames 200 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_small2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:linearize_kernel -s 3 -c 1 -o gpurun_out/prof_linearize_v2 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
