set -x
nproc; lscpu | head -20; free -g; nvidia-smi; nvidia-smi -q | grep -iE 'clocks|MHz' | head -30
cd tools/microbench && ./mb 29 2>&1 | tee ../../gpurun_out/mb29.txt
./mb 30 2>&1 | tail -8 | tee ../../gpurun_out/mb30.txt
