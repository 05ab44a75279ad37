# PCG vs Cholesky on the full c4 and the c3 (PCG by default) bench lines
for spec in "c4 pcg" "c4 cholesky" "c3 pcg" "c3 cholesky"; do
  set -- $spec
  timeout 1200 python bench.py --config $1 --solver $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/solver_$1_$2.log 2>&1; echo "$1 $2 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/solver_$1_$2.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$1 $2 step',d['ms_per_step'],'solve',r['solve_ms'],r.get('pcg_last_solve'))"
done
