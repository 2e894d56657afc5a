# round 2 (x): CELLS in-place accept (inplace_eff sweep) and odd stride for CELLS NEAREST
for ip in 0 50 70 85; do for cfg in "3" "5" "5 --W 24"; do
  echo "m ip=$ip | $(SPIN_INPLACE=$ip SPIN_LIB_PATH=abbuild/m/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2x.txt
done; done
for ip in 0 70; do for cfg in "5" "5 --W 24"; do
  echo "cn ip=$ip | $(SPIN_INPLACE=$ip SPIN_LIB_PATH=abbuild/cn/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2x.txt
done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "cells or fuzz or scale" 2>&1 | tail -4 >> gpurun_out/r2x.txt
cat gpurun_out/r2x.txt
