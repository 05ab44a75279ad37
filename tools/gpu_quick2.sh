for m in ${VARIANTS:-4 6 7 9}; do
PBA_LIN_VARIANT=$m timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_$m.log 2>&1; echo "variant $m rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/var_$m.log').read().strip().splitlines()[-1]);print('variant',$m,'step ms',d['ms_per_step'],'lin ms',d['roofline']['linearize_ms'],'frac',d['roofline']['frac'])"
done
