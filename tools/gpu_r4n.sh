# round 2 (4n): hi-only pre-pass (2 KB fragment halves per tile, K_pre) (y1) vs the final build (m)
for lib in m y1; do
  for cfg in "4" "4 --mode nearest"; do
    for sk in 0 2; do
    echo "$lib skip$sk cfg $cfg | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-150)" >> gpurun_out/r4n_ab.txt
    done
  done
done
SPIN_LIB_PATH=abbuild/y1/libspin.so python -m pytest tests -m gpu -q -x -k "not cells and not c3 and not c5" 2>&1 | tail -3 >> gpurun_out/r4n_ab.txt
cat gpurun_out/r4n_ab.txt
