set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo smoke=$?
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/val_pytest.log 2>&1; echo pytest=$?
timeout -s KILL 300 python tools/pfact_bench.py --nbmin 4096 16384 65536 131072 > gpurun_out/val_pfact_nbmin.jsonl 2>&1; echo pfact=$?
timeout -s KILL 600 python tools/dist_sweep.py 131072 512 1 1 "" "store_l=0" > gpurun_out/val_sw_storel.log 2>&1; echo sweep=$?
