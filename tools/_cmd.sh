o=gpurun_out/r01h; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
for c in c1 c4; do timeout 120 python bench.py --config $c --quick --steps 20 --proto ll >> $o/quick.jsonl 2>&1; done
for c in c2 c3; do timeout 120 python tools/trace.py --config $c --json $o/trace_$c.json > $o/trace_$c.log 2>&1; done
timeout 120 python tools/trace.py --config c1 --proto ll --json $o/trace_c1ll.json > $o/trace_c1ll.log 2>&1
bash tools/ab.sh "llb1:-DGC3_LL_BATCH=1;llb8:-DGC3_LL_BATCH=8" "c1 c4" "--proto ll" > $o/ab.txt 2>&1
bash tools/ab.sh "uc4:-DGC3_UNROLL_COPY=4;uc2:-DGC3_UNROLL_COPY=2" "c2 c2d c5ag" >> $o/ab.txt 2>&1
