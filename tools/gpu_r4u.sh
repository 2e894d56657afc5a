# round 2 (4u): dense_min sweep on the final build (measurement build, SPIN_DENSE_MIN)
for dm in 4 6 8 12 16; do
  for cfg in "4" "4 --mode nearest" "2" "6"; do
    echo "dense_min $dm cfg $cfg | $(SPIN_DENSE_MIN=$dm SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/r4u_ab.txt
  done
done
cat gpurun_out/r4u_ab.txt
