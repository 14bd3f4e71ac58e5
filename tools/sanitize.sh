#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_cases.py (one GPU;
# run under gpurun): gpurun -- 'bash tools/sanitize.sh r02'
tag=${1:-r02}
out=gpurun_out/$tag/sanitizer
mkdir -p $out
export GC3_TIMEOUT_MS=120000   # the tools slow every spin-wait down
for tool in memcheck racecheck synccheck initcheck; do
  for c in c1 c2 c3 c4df c1ll c1ll128 c5rs_tma; do
    timeout 900 compute-sanitizer --tool $tool --kernel-name kns=interp --print-limit 20 \
      python tools/sanitize_cases.py $c > $out/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|: ok' $out/${tool}_$c.log | tr '\n' ' ')" >> $out/summary.txt
  done
done
