#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py (every C-ABI entry point on small
# bands).  Run on the GPU box from the repo root:
#   bash tools/sanitize.sh [outdir]          (default gpurun_out/sanitize)
# (compute-sanitizer is closed on the gpurun pool of this build — the script exits
# after the plain run there; kept for boxes where the tool is allowed.)
# One log per tool; the last line of each is the tool's error summary.  initcheck and
# racecheck are restricted to this library's kernels (namespace cpm) — torch's and
# cub's own kernels are not ours to check.
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
python tools/sanitize_case.py > "$out/plain.log" 2>&1 || { echo "case fails without the sanitizer"; tail -5 "$out/plain.log"; exit 1; }
rc=0
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--kernel-name kns=cpm --racecheck-report all"
  [ "$tool" = initcheck ] && extra="--kernel-name kns=cpm --track-unused-memory no"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 40 \
    --log-file "$out/$tool.log" python tools/sanitize_case.py > "$out/$tool.stdout" 2>&1
  r=$?
  echo "$tool exit $r: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$out/$tool.log" | tail -1)"
  [ $r -ne 0 ] && rc=1
done
exit $rc
