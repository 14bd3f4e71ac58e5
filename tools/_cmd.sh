o=gpurun_out/r01o; mkdir -p $o
GC3_TMA=7 timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
bash tools/envsweep.sh "c2 c2d c5ag c3 c4 c1" "GC3_TMA=3;GC3_TMA=7;GC3_TMA=7 GC3_UNIT_WARPS=8" > $o/env.txt 2>&1
GC3_TMA=7 timeout 120 python tools/trace.py --config c2 --json $o/trace_c2.json > $o/trace_c2.log 2>&1
