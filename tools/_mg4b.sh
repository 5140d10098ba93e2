set -x
timeout -s KILL 1200 python -m pytest tests/test_multi_gpu.py -q -k "peer or 1x4 or 4gpu" > gpurun_out/mg4b_pytest.log 2>&1; echo pytest=$?
