# round-1 profile captures (one GPU): full-set CVP forward/backward at 16 views,
# then the launch list + DRAM bytes of one bench step (c3, 496 views)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -c 1 -o gpurun_out/prof_f python tools/prof_cvp.py --views 16 > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cvp_brick -s 1 -c 1 -o gpurun_out/prof_b python tools/prof_cvp.py --views 16 > gpurun_out/ncu_b.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --cgls-iters 0 > gpurun_out/bench_ncu.log 2>&1
