# round 2 (5d): knob re-checks on the final build (C4): e1 two candidates per lane in the BRUTE accept pass,
# e2 no dense-tile queue, e3 lane 0 alone polls the tile barrier, e4 / e5 image stride residue 9 / 5
for lib in paper_1811_00901_b200 abbuild/e1 abbuild/e2 abbuild/e3 abbuild/e4 abbuild/e5; do
  for cfg in "4" "4 --mode nearest"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r5d_ab.txt
  done
done
cat gpurun_out/r5d_ab.txt
