# round 2 (5b): knob re-checks on the final build: two live rows per dense-walk step (d2), tensor-core batch 2 (b2)
for lib in paper_1811_00901_b200 abbuild/d2 abbuild/b2; do
  for cfg in "4" "4 --mode nearest" "2"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r5b_ab.txt
  done
done
cat gpurun_out/r5b_ab.txt
