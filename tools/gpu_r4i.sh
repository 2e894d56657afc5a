# round 2 (4i): candidates counted per tile (k1) or per accept pass (k0), both with the host-side bin constants
for lib in k0 k1; do
  for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6" "3" "5" "5 --W 24"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/r4i_ab.txt
  done
done
cat gpurun_out/r4i_ab.txt
