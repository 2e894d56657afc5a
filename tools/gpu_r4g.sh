# round 2 (4g): CELLS accept passes with pinned shared-window addresses + one clamp before rsqrt (c3) vs c2
for lib in c2 c3; do
  for cfg in "3" "5" "5 --W 24" "6"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4g_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/c3/libspin.so python -m pytest tests -m gpu -q -x -k "cells or c3 or c5 or fuzz or nearest or p6" 2>&1 | tail -5 >> gpurun_out/r4g_ab.txt
cat gpurun_out/r4g_ab.txt
