#!/bin/bash
# One GPU-box pass (run under gpurun): parity tests, smoke, per-config quick timings, the default
# bench line, the ncu launch list and one `ncu --set full` capture of the interpreter kernel.
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh [tag] [configs] [full-capture-config]'
tag=${1:-r01}
configs=${2:-"c1 c2 c2d c3 c4 c5ag c5rs"}
capcfg=${3:-c2}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for c in $configs; do
  timeout 180 python bench.py --config $c --quick --steps 20 >> $out/quick.jsonl 2>>$out/quick.err
done
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$capcfg.csv \
  python bench.py --config $capcfg --steps 4 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp -s 3 -c 1 \
  -o $out/prof_$capcfg python bench.py --config $capcfg --quick --steps 1 --warmup 3 > $out/ncu_full.log 2>&1
echo done
