# ncu --set full of the c3 CVP forward and backward (all 496 views, brick
# shape fixed so no tuning launches are captured), one report each, plus the
# per-kernel summary and per-source-line hot spots, and the launch list of one
# bench step.  usage: bash tools/prof_cvp_pair.sh TAG   (outputs gpurun_out/*_TAG*)
tag=${1:-cur}
mkdir -p gpurun_out
export CVPB_CVP_SHAPE=${CVPB_CVP_SHAPE:-0}
for dir in fwd bwd; do
    skip=0; [ $dir = bwd ] && skip=1
    ncu --set full --clock-control none --import-source on -k regex:cvp_brick -s $skip -c 1 \
        -o gpurun_out/prof_${tag}_$dir -f python tools/prof_cvp.py --views 496 > gpurun_out/ncu_${tag}_$dir.log 2>&1
    python tools/ncu_summary.py gpurun_out/prof_${tag}_$dir.ncu-rep > gpurun_out/ncu_${tag}_${dir}_summary.txt 2>&1
    python tools/ncu_lines.py gpurun_out/prof_${tag}_$dir.ncu-rep cvp_brick 60 > gpurun_out/ncu_${tag}_${dir}_lines.txt 2>&1
done
unset CVPB_CVP_SHAPE
if [ "${LAUNCHES:-1}" = 1 ]; then
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-other-precision \
    --cgls-iters 0 > gpurun_out/bench_ncu_${tag}.log 2>&1
fi
