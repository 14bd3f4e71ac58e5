o=gpurun_out/r01ah; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "special_values or dtypes or allreduce_f32" > $o/pytest_sel.log 2>&1; echo "rc=$?" >> $o/pytest_sel.log
GC3_TMA=3 timeout 900 python -m pytest tests -m gpu -q -k "special_values" > $o/pytest_sel_notma8.log 2>&1; echo "rc=$?" >> $o/pytest_sel_notma8.log
bash tools/envsweep.sh "c3 c4 c5rs" "GC3_TMA=11;GC3_TMA=3" > $o/env.txt 2>&1
bash tools/envsweep.sh "c2" "GC3_UNIT_WARPS=2;GC3_UNIT_WARPS=4;GC3_WQ_ITEMS=5" >> $o/env.txt 2>&1
