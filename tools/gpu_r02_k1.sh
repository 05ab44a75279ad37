# after a K1 change: GPU suite, default bench, launch list (c4/200) and one full ncu capture of K1 on the full c4 bench
timeout 1500 python -m pytest tests -m gpu -q -x --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_default.log').read().strip().splitlines()[-1]);print('step',d['ms_per_step'],'lin',d['roofline']['linearize_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['ms_per_step'],'api',d.get('e2e_api',{}).get('seconds'))"
CMD2="python bench.py --config c4 --frames 200 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-api"
timeout 600 $CMD2 > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD2 > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
CMD3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-api"
timeout 900 $CMD3 > gpurun_out/plain_full.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:linearize_kernel -s 4 -c 1 -o gpurun_out/prof_lin_c4full -f $CMD3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
