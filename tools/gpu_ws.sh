PBA_LIN_VARIANT=30 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=short -x > gpurun_out/pytest_ws.log 2>&1; echo "pytest ws rc=$?"; tail -15 gpurun_out/pytest_ws.log
VARIANTS="4 30 31 32 33" bash tools/gpu_quick3.sh
