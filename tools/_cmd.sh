o=gpurun_out/r01aa; mkdir -p $o
bash tools/envsweep.sh "c1 c5ag c5rs c4" "GC3_TMA_MIN=0;GC3_TMA_MIN=16384;GC3_TMA_MIN=32768;GC3_TMA_MIN=65536" > $o/env.txt 2>&1
timeout 600 python bench.py --config c4 --sweep --sweep-min 1024 --sweep-max 16777216 --sweep-protos simple --steps 20 > $o/sweep.jsonl 2>&1
GC3_TMA_MIN=0 timeout 600 python bench.py --config c4 --sweep --sweep-min 1024 --sweep-max 16777216 --sweep-protos simple --steps 20 > $o/sweep0.jsonl 2>&1
