mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -c 1 -o gpurun_out/prof_f python tools/prof_cvp.py --views 16 > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -s 1 -c 1 -o gpurun_out/prof_b python tools/prof_cvp.py --views 16 > gpurun_out/ncu_b.log 2>&1
