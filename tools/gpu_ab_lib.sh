# A/B of two builds of the library (PBA_LIBRARY) on one config, alternating, one process per run
run() { # tag lib
  PBA_LIBRARY=$2 timeout 900 python bench.py --config ${CFG:-c4} ${FRAMES:+--frames $FRAMES} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/ablib_$1.log 2>&1; echo "$1 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/ablib_$1.log').read().strip().splitlines()[-1]);print('$1','step ms',round(d['ms_per_step'],3),'lin ms',round(d['roofline']['linearize_ms'],3))"
}
A=${A:-gpurun_variants/libA.so}; B=${B:-paper_2303_16878_b200/_lib/libpba_b200.so}
for i in 1 2; do run A$i $A; run B$i $B; done
