# round 2 (4w): CELLS group size on the final build (measurement build, SPIN_DEBUG_G)
for g in 8 16 32; do
  for cfg in "3" "5" "5 --W 24"; do
    echo "G $g cfg $cfg | $(SPIN_DEBUG_G=$g SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r4w_ab.txt
  done
done
cat gpurun_out/r4w_ab.txt
