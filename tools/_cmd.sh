o=gpurun_out/r01g; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
for c in c1 c2 c3 c4 c5rs c5ag c2d; do timeout 120 python bench.py --config $c --quick --steps 20 >> $o/quick.jsonl 2>&1; done
for c in c1 c4; do timeout 120 python bench.py --config $c --quick --steps 20 --proto ll >> $o/quick.jsonl 2>&1; done
for c in c1 c2; do timeout 120 python tools/trace.py --config $c --json $o/trace_$c.json > $o/trace_$c.log 2>&1; done
timeout 120 python tools/trace.py --config c1 --proto ll --json $o/trace_c1ll.json > $o/trace_c1ll.log 2>&1
timeout 900 python bench.py --config c4 --sweep --sweep-min 1024 --sweep-max 1073741824 --steps 20 > $o/sweep_c4.jsonl 2>&1
bash tools/ab.sh "u2:-DGC3_UNROLL=2;uc4:-DGC3_UNROLL_COPY=4" "c1 c2 c3 c4" > $o/ab.txt 2>&1
