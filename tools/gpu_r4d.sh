# round 2 (4d): fragments from L2 straight into registers (FRAGREG) vs the bulk-copy build (p1)
for lib in p1 r1; do
  for cfg in "4" "4 --mode nearest"; do
    for sk in 0 2; do
    echo "$lib skip$sk cfg $cfg | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4d_ab.txt
    done
  done
done
SPIN_LIB_PATH=abbuild/r1/libspin.so python -m pytest tests -m gpu -q -x -k "not cells and not c3 and not c5" 2>&1 | tail -5 >> gpurun_out/r4d_ab.txt
cat gpurun_out/r4d_ab.txt
