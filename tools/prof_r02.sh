# round-2 ncu captures (one GPU): CVP forward + backward, c3, all 496 views,
# brick shape fixed (no tuning launches), full section set
mkdir -p gpurun_out
export CVPB_CVP_SHAPE=${CVPB_CVP_SHAPE:-0}
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -c 2 -o gpurun_out/prof_r02 -f \
    python tools/prof_cvp.py --views 496 > gpurun_out/ncu_r02.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02.ncu-rep
