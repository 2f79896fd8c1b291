mkdir -p gpurun_out
bash tools/ab.sh "unr m" "c3 c4 c2" 128 > gpurun_out/ab3.txt 2>&1
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests3.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests3.log
python bench.py > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
python tools/bench_configs.py > gpurun_out/configs_m.txt 2>&1
bash tools/prof_cvp_pair.sh r02m
mkdir -p /tmp/ncurep; mv gpurun_out/*.ncu-rep /tmp/ncurep/ 2>/dev/null
du -sh gpurun_out
cat gpurun_out/ab3.txt; tail -2 gpurun_out/gpu_tests3.log
