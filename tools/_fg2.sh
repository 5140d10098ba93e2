set -x
timeout -s KILL 900 python -m pytest tests/test_multi_gpu.py -q -x -k "2x1 or gathered or peer" > gpurun_out/fg2_pytest.log 2>&1; echo pytest=$?
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/dist_sweep.py 131072 512 2 1 "" "fact_gather_ms=100000" "fact_gather=32768,fact_gather_ms=100000" > gpurun_out/fg2_sweep.log 2>&1; echo sweep=$?
