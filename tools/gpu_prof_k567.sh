# ncu captures of the preprocessing kernels (K5 overlap, K6 pyramid, K7 decode)
timeout 300 python tools/pyramid_bench.py --frames 64 > gpurun_out/pyr_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"normals_kernel|moment_colscan|moment_rowscan|downscale_kernel" -c 4 -o gpurun_out/prof_k6 -f python tools/pyramid_bench.py --frames 64 --reps 1 > gpurun_out/ncu_k6.log 2>&1; echo "k6 rc=$?"
timeout 300 python tools/dataset_bench.py --frames 64 --host-frames 1 > gpurun_out/ds_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:decode_kernel -c 2 -o gpurun_out/prof_k7 -f python tools/dataset_bench.py --frames 64 --host-frames 1 > gpurun_out/ncu_k7.log 2>&1; echo "k7 rc=$?"
CMD="python bench.py --config c4 --frames 200 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_k5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:overlap_kernel -c 1 -o gpurun_out/prof_k5 -f $CMD > gpurun_out/ncu_k5.log 2>&1; echo "k5 rc=$?"
