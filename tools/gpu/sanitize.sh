# ONE compute-sanitizer tool per gpurun call (pool rule), every case of
# tools/sanitize_cases.py in one process.   usage: bash tools/gpu/sanitize.sh TOOL
t=${1:-memcheck}
extra=""
[ "$t" = "racecheck" ] && extra="--racecheck-report hazard"
mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool $t $extra --error-exitcode 9 python tools/sanitize_cases.py all \
  > gpurun_out/san/$t.log 2>&1
echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$t.log | tail -1)" | tee -a gpurun_out/san/summary.txt
