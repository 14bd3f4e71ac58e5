o=gpurun_out/r01k; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
for c in c1 c2 c3 c4 c5rs c5ag c2d; do timeout 120 python bench.py --config $c --quick --steps 20 >> $o/quick.jsonl 2>&1; done
bash tools/envsweep.sh "c3 c4 c5rs c1" "GC3_TMA=1;GC3_UNIT_WARPS=2;GC3_UNIT_WARPS=2 GC3_TMA=1" > $o/env.txt 2>&1
bash tools/envsweep.sh "c2 c2d c5ag" "GC3_UNIT_WARPS=2;GC3_TMA=0" >> $o/env.txt 2>&1
