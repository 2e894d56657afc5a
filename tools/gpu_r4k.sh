# round 2 (4k): CELLS bounding-box cull of centre batches with contiguous warp tiles (u1) vs the default build
for lib in paper_1811_00901_b200 abbuild/u1; do
  for cfg in "3" "5" "5 --W 24" "3 --mode nearest" "5 --mode bilinear"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4k_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/u1/libspin.so python -m pytest tests -m gpu -q -x -k "cells or c3 or c5 or fuzz" 2>&1 | tail -5 >> gpurun_out/r4k_ab.txt
cat gpurun_out/r4k_ab.txt
