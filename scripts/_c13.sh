mkdir -p gpurun_out/c13
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4 or config3 or golden or corpus or dequant" > gpurun_out/c13/pytest.log 2>&1; echo rc=$? >> gpurun_out/c13/pytest.log
timeout 200 python scripts/decode_bench.py > gpurun_out/c13/decode.txt 2>&1
