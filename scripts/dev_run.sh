mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "dequant" > gpurun_out/abl/deq_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/deq_tests.txt
