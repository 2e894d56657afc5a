# round 2 (4c): half-size fragment copy (row blocks 4-7 reuse 0-3), filter only: does the
# BRUTE filter follow the L2 -> SM bytes?
for lib in m0 x2; do
  for cfg in "4" "4 --mode nearest"; do
    for sk in 2 1; do
    echo "$lib skip$sk cfg $cfg | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4c_ab.txt
    done
  done
done
cat gpurun_out/r4c_ab.txt
