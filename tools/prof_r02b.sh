# round-2 evidence pass (one GPU):
#  1. shared-memory atomic peak (SURVEY 8d secondary roof)
#  2. ncu --set full of the CVP forward + backward at c3 (all 496 views, fixed brick shape)
#  3. ncu --set full of the TT pair (c3 geometry, 16 views) and Siddon-K (c2, 16 views)
#  4. the launch list + DRAM bytes of one bench step (c3, 496 views)
mkdir -p gpurun_out build
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/smem_atomic_peak tools/smem_atomic_peak.cu && \
    ./build/smem_atomic_peak > gpurun_out/smem_atomic_peak.json
export CVPB_CVP_SHAPE=${CVPB_CVP_SHAPE:-0}
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -c 2 -o gpurun_out/prof_r02 -f \
    python tools/prof_cvp.py --views 496 > gpurun_out/ncu_r02.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02.ncu-rep > gpurun_out/ncu_r02_summary.txt 2>&1
unset CVPB_CVP_SHAPE
ncu --set full --clock-control none --import-source on -k regex:tt_ -c 2 -o gpurun_out/prof_tt_r02 -f \
    python tools/prof_tt.py > gpurun_out/ncu_tt_r02.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_tt_r02.ncu-rep > gpurun_out/ncu_tt_r02_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:siddon -c 3 -o gpurun_out/prof_siddon_r02 -f \
    python tools/prof_siddon.py > gpurun_out/ncu_siddon_r02.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_siddon_r02.ncu-rep > gpurun_out/ncu_siddon_r02_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    --cgls-iters 0 > gpurun_out/bench_ncu_r02.log 2>&1
