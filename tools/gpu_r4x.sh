# round 2 (4x): CELLS cell edge R / k on the final build (measurement build, SPIN_DEBUG_CELLS_PER_R)
for k in 6 8 10 12; do
  for cfg in "3" "5" "5 --W 24"; do
    echo "cells_per_R $k cfg $cfg | $(SPIN_DEBUG_CELLS_PER_R=$k SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r4x_ab.txt
  done
done
cat gpurun_out/r4x_ab.txt
