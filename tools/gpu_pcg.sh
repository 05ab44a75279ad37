timeout 600 python -m pytest tests/test_gpu_pcg.py -q -x > gpurun_out/pcg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pcg_tests.log
timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline --solver pcg > gpurun_out/pcg_c4_200.log 2>&1; echo "c4/200 pcg rc=$?"
timeout 900 python bench.py --config c4 --frames 200 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/chol_c4_200.log 2>&1; echo "c4/200 chol rc=$?"
for f in pcg_c4_200 chol_c4_200; do python -c "import json;d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$f',d['ms_per_step'],r['solve_ms'],r.get('pcg_last_solve'))"; done
