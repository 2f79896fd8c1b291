#!/bin/bash
# The paper's timing protocol (mean P / BP time inside CGLS on
# U[0,1) data) through the cbctproj-compatible CLI, for the paper presets.
mkdir -p gpurun_out
P="python -m paper_2110_09841_b200 bench --iterations 4"
$P --preset long2010 --csv gpurun_out/bench_long2010_cvp.csv
$P --preset long2010 --relaxed --csv gpurun_out/bench_long2010_relaxed.csv
$P --preset long2010 --projector tt --csv gpurun_out/bench_long2010_tt.csv
$P --preset pfeiffer2021 --csv gpurun_out/bench_pfeiffer2021_cvp.csv
$P --preset pfeiffer2021 --projector siddon --siddon-k 8 --iterations 2 --csv gpurun_out/bench_pfeiffer2021_siddon8.csv
