# final-kernel evidence pass (one GPU): parity tables and compute-sanitizer
mkdir -p gpurun_out
timeout 900 python tools/parity_report.py > gpurun_out/parity_final.md 2>&1
timeout 1200 python tools/config_parity_report.py > gpurun_out/config_parity_final.md 2>&1
for t in memcheck racecheck synccheck; do
  echo "## $t"; timeout 900 compute-sanitizer --tool $t python tools/sanitize_case.py 2>&1 | tail -6
done > gpurun_out/sanitizer_final.txt
