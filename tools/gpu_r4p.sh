# round 2 (4p): ablations of the BRUTE pre-pass (measurement builds, wrong images, SPIN_DEBUG_SKIP=2):
# a8 no tile ever has a candidate (the pure pre-pass pipeline), a9 + no HMMAs, a10 + no fragment copy,
# a12 + no AND chain, a14 + no copy and no AND chain
for lib in m a8 a9 a10 a12 a14; do
  for cfg in "4" "2"; do
    echo "$lib skip2 cfg $cfg | $(SPIN_DEBUG_SKIP=2 SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/r4p_ab.txt
  done
done
cat gpurun_out/r4p_ab.txt
