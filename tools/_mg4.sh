set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout -s KILL 180 $TR --master-port 29521 tools/dist_hpl.py 2048 128 2 2 42 --oracle > gpurun_out/mg4_canary22.log 2>&1; echo canary22=$?
timeout -s KILL 900 python -m pytest tests/test_multi_gpu.py -x -q -k "4gpu or peer or 1x4" > gpurun_out/mg4_pytest.log 2>&1; echo pytest=$?
timeout -s KILL 1200 $TR --master-port 29522 bench.py --gpus 4 --steps 1 --warmup 3 > gpurun_out/mg4_bench.json 2> gpurun_out/mg4_bench.err; echo bench=$?
