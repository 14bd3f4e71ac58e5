#!/bin/bash
# End-of-round evidence pass (run under gpurun, 1 GPU):
#   gpurun --timeout 3000 -- 'bash tools/final_round.sh r01z'
# parity tests, smoke, every config's timing, the C4 size sweep (Simple and LL), the default bench
# line and the reference arm, ncu launch lists + full captures (headline C2, C4 per protocol, C3),
# summarised on the box into gpurun_out/<tag>/profiles (merge with tools/ncu_summary.py --merge).
tag=${1:-final}
o=gpurun_out/$tag
mkdir -p $o
nvidia-smi > $o/nvidia-smi.txt 2>&1
lscpu > $o/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $o/smoke.log 2>&1; echo "rc=$?" >> $o/smoke.log
for c in c1 c1ap c2 c2d c3 c4 c4auto c5ag c5rs; do timeout 180 python bench.py --config $c --quick --steps 20 >> $o/quick.jsonl 2>>$o/quick.err; done
for c in c1 c4; do timeout 180 python bench.py --config $c --quick --steps 20 --proto ll >> $o/quick.jsonl 2>>$o/quick.err; done
timeout 900 python bench.py --config c4 --sweep --steps 20 --graph > $o/sweep_c4.jsonl 2> $o/sweep_c4.err
timeout 600 python bench.py --config c1 --sweep --steps 20 --sweep-max 268435456 --graph > $o/sweep_c1.jsonl 2> $o/sweep_c1.err
timeout 600 python bench.py --config c4 --sweep --builtin --sweep-max 16777216 --steps 20 --graph > $o/sweep_builtin.jsonl 2> $o/sweep_builtin.err
timeout 600 python bench.py > $o/bench.json 2> $o/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.json 2> $o/bench_ref.err
bash tools/gpu_ncu.sh $tag "c2 c3 c4 c5rs c5ag c1" > /dev/null 2>&1
# LL capture of C4 under its own name
mkdir -p $o/ll
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_c4ll.csv \
  python bench.py --config c4 --quick --steps 4 --warmup 3 --proto ll > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp -s 3 -c 1 \
  -o $o/prof_c4ll python bench.py --config c4 --quick --steps 1 --warmup 3 --proto ll > $o/ncu_full_c4ll.log 2>&1
python tools/ncu_summary.py $tag c4ll ring_ar_8_ch8_inst4.ll 67108864 --out $o/profiles > /dev/null 2>> $o/summary.err
find $o -size +6M -name '*.ncu-rep' -delete
echo done
