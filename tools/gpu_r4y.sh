# round 2 (4y): CELLS accept passes gathering the centre from component arrays (z1), plus an odd image
# stride for NEAREST too (z2), vs the committed build
for lib in paper_1811_00901_b200 abbuild/z1 abbuild/z2; do
  for cfg in "3" "5" "5 --W 24" "3 --mode nearest"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r4y_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/z2/libspin.so python -m pytest tests -m gpu -q -x -k "cells or c3 or c5 or fuzz" 2>&1 | tail -2 >> gpurun_out/r4y_ab.txt
cat gpurun_out/r4y_ab.txt
