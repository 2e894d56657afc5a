# round 2 (5a): BILINEAR W constants from the host + pinned CELLS image stride (t1) vs the committed build
for lib in paper_1811_00901_b200 abbuild/t1; do
  for cfg in "3" "5" "5 --W 24" "4" "2" "3 --mode nearest" "5 --mode bilinear"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r5a_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/t1/libspin.so python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/r5a_ab.txt
cat gpurun_out/r5a_ab.txt
