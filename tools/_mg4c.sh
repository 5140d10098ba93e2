set -x
timeout -s KILL 1200 python -m pytest tests/test_multi_gpu.py -q -k "4gpu or peer or 1x4 or gathered" > gpurun_out/mg4c_pytest.log 2>&1; echo pytest=$?
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --steps 1 --warmup 3 > gpurun_out/mg4c_bench.json 2> gpurun_out/mg4c_bench.err; echo bench=$?
