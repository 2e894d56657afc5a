# round 2 (4q): what a tile with a candidate costs in the filter (SPIN_DEBUG_SKIP=2): a32 no point staging,
# a64 no mask pass, a96 neither (= a8 plus the vote's branch)
for lib in m a8 a32 a64 a96; do
  for cfg in "4" "4 --mode nearest"; do
    echo "$lib skip2 cfg $cfg | $(SPIN_DEBUG_SKIP=2 SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/r4q_ab.txt
  done
done
cat gpurun_out/r4q_ab.txt
