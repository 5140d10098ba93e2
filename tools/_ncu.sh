set -x
timeout -s KILL 200 python tools/ncu_dgemm.py 32768 > gpurun_out/ncu_plain.log 2>&1; echo plain=$?
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 1 -c 1 -f -o gpurun_out/prof_dgemm_32k python tools/ncu_dgemm.py 32768 > gpurun_out/ncu_run.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_dgemm_32k.ncu-rep --page raw --csv > gpurun_out/prof_dgemm_32k_raw.csv 2>&1
ncu -i gpurun_out/prof_dgemm_32k.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_dgemm_32k_sass.csv 2>&1
ls -la gpurun_out/
