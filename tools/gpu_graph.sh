# graph construction on the device: edge-list parity tests + c4 graph build time
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "build_graph" > gpurun_out/pt_graph.log 2>&1; echo "graph tests rc=$?"; tail -2 gpurun_out/pt_graph.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/graph_bench.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/graph_bench.log').read().strip().splitlines()[-1]);print('graph_seconds',d['config']['graph_seconds'],'setup',d['config']['setup_seconds'],'pairs',d['config']['pairs'])"
