# round 2 (4b): A/B of the CELLS half-tile compaction (h0/h1), the pinned dense-walk image
# address (m0/p1) and the half-size fragment copy experiment (x2, filter only: is the BRUTE
# filter bound by L2 -> SM bandwidth?)
for lib in h0 h1; do
  for cfg in "3" "5" "5 --W 24"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4b_ab.txt
  done
done
for lib in m0 p1; do
  for cfg in "4" "4 --mode nearest" "2"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4b_ab.txt
  done
done
for lib in m0 x2; do
  for cfg in "4" "2"; do
    echo "$lib skip2 cfg $cfg | $(SPIN_DEBUG_SKIP=2 SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4b_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/h1/libspin.so python -m pytest tests -m gpu -q -k "cells or c3 or c5 or fuzz" 2>&1 | tail -5 >> gpurun_out/r4b_ab.txt
cat gpurun_out/r4b_ab.txt
