o=gpurun_out/r01q; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
bash tools/envsweep.sh "c2 c2d c5ag c3 c4 c5rs c1" "GC3_UNIT_WARPS=4;GC3_UNIT_WARPS=2;GC3_UNIT_WARPS=1" > $o/env.txt 2>&1
bash tools/envsweep.sh "c2 c5ag c3 c4" "GC3_TILE_BYTES=32768;GC3_TILE_BYTES=65536;GC3_UNIT_WARPS=2 GC3_TILE_BYTES=32768;GC3_UNIT_WARPS=2 GC3_MAX_LANES=128" >> $o/env.txt 2>&1
