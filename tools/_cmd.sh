o=gpurun_out/r01p; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
bash tools/envsweep.sh "c2 c2d c5ag c3 c4 c5rs" "GC3_TAPER=1;GC3_TAPER=0" > $o/env.txt 2>&1
timeout 120 python tools/trace.py --config c2 --json $o/trace_c2.json > $o/trace_c2.log 2>&1
