# one-GPU round pass: parity suite, bench line, all-config table, ncu of the
# c3 CVP pair (reports summarised to text, the .ncu-rep files moved out of
# gpurun_out/ so the copy-back stays under its 64 MiB cap)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/bench_configs.py > gpurun_out/configs.txt 2>&1
bash tools/prof_cvp_pair.sh final
mkdir -p /tmp/ncurep; mv gpurun_out/*.ncu-rep /tmp/ncurep/ 2>/dev/null
tail -2 gpurun_out/gpu_tests.log
