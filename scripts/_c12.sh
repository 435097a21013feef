mkdir -p gpurun_out/c12
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4 or config3 or smoke or corpus" > gpurun_out/c12/pytest.log 2>&1; echo rc=$? >> gpurun_out/c12/pytest.log
timeout 200 python scripts/decode_bench.py > gpurun_out/c12/decode.txt 2>&1
APMM_LIB=$PWD/devlib/libapmm_old.so timeout 200 python scripts/decode_bench.py > gpurun_out/c12/decode_old.txt 2>&1
