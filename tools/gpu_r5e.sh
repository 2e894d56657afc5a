# round 2 (5e): knob re-checks for the 768-thread launches (C2, P6): f1 two live rows per dense-walk step,
# f2 no pre-pass phase, f3 two candidates per lane in the accept pass
for lib in paper_1811_00901_b200 abbuild/f1 abbuild/f2 abbuild/f3; do
  for cfg in "2" "2 --mode nearest" "6"; do
    for rep in 1 2; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r5e_ab.txt
    done
  done
done
cat gpurun_out/r5e_ab.txt
