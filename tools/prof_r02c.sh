# round-2: ncu --set full of the CVP backward alone at c3 (496 views, fixed shape)
mkdir -p gpurun_out
export CVPB_CVP_SHAPE=${CVPB_CVP_SHAPE:-0}
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -s 1 -c 1 -o gpurun_out/prof_r02_bwd -f \
    python tools/prof_cvp.py --views 496 > gpurun_out/ncu_r02_bwd.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02_bwd.ncu-rep > gpurun_out/ncu_r02_bwd_summary.txt 2>&1
