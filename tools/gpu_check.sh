#!/bin/bash
# Quick GPU pass (run under gpurun): parity tests, smoke, per-config quick timings with and without
# the dataflow executor (GC3_DF=0 / default).
#   gpurun --timeout 1800 -- 'bash tools/gpu_check.sh <tag> ["configs"] [pytest-args]'
tag=${1:-r02}
configs=${2:-"c1 c2 c3 c4 c5ag c5rs"}
ptargs=${3:-"tests -m gpu -x -q"}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest $ptargs > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for c in $configs; do
  for df in 0 1; do
    GC3_DF=$df timeout 180 python bench.py --config $c --quick --steps 20 | sed "s/^/{\"df\": $df, \"r\": /; s/\$/}/" >> $out/quick.jsonl 2>>$out/quick.err
  done
done
echo done
