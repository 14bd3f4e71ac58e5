o=gpurun_out/r01ak; mkdir -p $o
GC3_BUILD_TAG=_f32 GC3_LIB_OUT=/tmp/libgc3_f32.so GC3_NVCC_DEFS="-DGC3_F32_BULKADD=1" python -m paper_2201_11840_b200.build > /tmp/b.log 2>&1
GC3_LIB_PATH=/tmp/libgc3_f32.so timeout 600 python -m pytest tests -m gpu -q -k "special_values" > $o/f32.log 2>&1; echo "rc=$?" >> $o/f32.log
timeout 600 python -m pytest tests -m gpu -q -k "special_values" > $o/default.log 2>&1; echo "rc=$?" >> $o/default.log
GC3_TMA=3 timeout 600 python -m pytest tests -m gpu -q -k "special_values" > $o/tma3.log 2>&1; echo "rc=$?" >> $o/tma3.log
