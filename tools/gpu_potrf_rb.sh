# potrf trailing update in registers (PBA_POTRF_RB=1, default) vs shared memory (0)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cholesky or solve or trace" > gpurun_out/pt_rb.log 2>&1; echo "solver tests rc=$?"; tail -1 gpurun_out/pt_rb.log
for rb in 1 0; do
  echo "RB=$rb"
  PBA_POTRF_RB=$rb timeout 300 python tools/solve_bench.py --dim 5994 --band 126 2>&1 | tail -2
  PBA_POTRF_RB=$rb timeout 300 python tools/solve_bench.py --dim 594 2>&1 | tail -2
  PBA_POTRF_RB=$rb timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rb_c2_$rb.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/rb_c2_$rb.log').read().strip().splitlines()[-1]);print('c2 step',round(d['ms_per_step'],3),'solve',d['roofline']['solve_ms'])"
  PBA_POTRF_RB=$rb timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rb_c4_$rb.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/rb_c4_$rb.log').read().strip().splitlines()[-1]);print('c4 step',round(d['ms_per_step'],3),'solve',d['roofline']['solve_ms'])"
done
