mkdir -p gpurun_out
BSG_P23=1 BSG_P23_LAG=2 ncu --set full --clock-control none --import-source on -k regex:k_part23 -s 1 -c 1 -o gpurun_out/prof_p23 python tools/run_once.py 29 2 1 > gpurun_out/prof_p23.log 2>&1
BSG_P23=0 ncu --set full --clock-control none --import-source on -k regex:"k_part2|k_part1" -s 2 -c 2 -o gpurun_out/prof_p2 python tools/run_once.py 29 2 1 > gpurun_out/prof_p2.log 2>&1
ls -la gpurun_out
