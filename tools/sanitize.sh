#!/bin/sh
# compute-sanitizer over the TMA / mbarrier kernels (tools/sanitize_cases.py):
# racecheck (shared-memory hazards incl. the TMA ring), synccheck (barrier
# misuse), memcheck (out-of-bounds / misaligned global and shared accesses).
# Logs go to gpurun_out/sanitize/; the summaries are copied into profiles/.
# The persistent kernels' dependency-wait timeout is raised because the
# tools slow every kernel down by orders of magnitude.
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
export HRT_PERSIST_TIMEOUT_S=600
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  for c in wave2 wave2_narrow wave tma4 tma volume_tma; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
      > "$OUT/${tool}_$c.log" 2>&1
    echo "$tool $c rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|case ' "$OUT/${tool}_$c.log" | tr '\n' ' ')" \
      | tee -a "$OUT/summary.txt"
  done
done
