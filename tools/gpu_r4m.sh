# round 2 (4m): A/B of CELLS knobs on the trimmed accept path (v1: halves for BILINEAR too, v2: one candidate
# per lane for BILINEAR, v3: two for NEAREST) and of quarter-tile dealing in phase 2 (w1) vs the default build
for lib in paper_1811_00901_b200 abbuild/v1 abbuild/v2 abbuild/v3; do
  for cfg in "3" "5" "5 --W 24"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-70)" >> gpurun_out/r4m_ab.txt
  done
done
for lib in paper_1811_00901_b200 abbuild/w1; do
  for cfg in "2" "2 --mode nearest" "6" "4" "1"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-70)" >> gpurun_out/r4m_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/w1/libspin.so python -m pytest tests -m gpu -q -x -k "not cells and not c3 and not c5" 2>&1 | tail -3 >> gpurun_out/r4m_ab.txt
cat gpurun_out/r4m_ab.txt
