#!/bin/bash
# ncu launch list + one full capture per config (run under gpurun; 1 GPU). Summaries are written on
# the box (gpurun_out/<tag>/profiles; merge with `python tools/ncu_summary.py --merge ...`); only
# small reports travel back.
#   gpurun -- 'bash tools/gpu_ncu.sh <tag> "c3 c4 c5rs" [extra bench args]'
tag=${1:-r01}
configs=${2:-"c3 c4"}
extra=${3:-}
out=gpurun_out/$tag
mkdir -p $out
declare -A IR=([c1]=ring_ar_8_ch1 [c2]=twostep_a2a_2x4 [c2d]=twostep_a2a_1x8 [c3]=hier_ar_2x4_par1 [c4]=ring_ar_8_ch8_inst4 [c5ag]=ring_ag_8 [c5rs]=ring_rs_8)
declare -A BYTES=([c1]=4194304 [c2]=67108864 [c2d]=67108864 [c3]=268435456 [c4]=67108864 [c5ag]=67108864 [c5rs]=67108864)
for c in $configs; do
  b=${BYTES[$c]}
  for a in $extra; do case $a in --bytes=*) b=${a#--bytes=};; esac; done
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$c.csv \
    python bench.py --config $c --quick --steps 4 --warmup 3 $extra > $out/ncu_launch_$c.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp -s 3 -c 1 \
    -o $out/prof_$c python bench.py --config $c --quick --steps 1 --warmup 3 $extra > $out/ncu_full_$c.log 2>&1
  timeout 120 python bench.py --config $c --quick --steps 20 $extra >> $out/quick.jsonl 2>>$out/quick.err
  python tools/ncu_summary.py $tag $c ${IR[$c]} $b --out $out/profiles > /dev/null 2>> $out/summary.err
done
du -sh $out/* > $out/sizes.txt 2>&1
find $out -size +6M -name '*.ncu-rep' -delete
echo done
