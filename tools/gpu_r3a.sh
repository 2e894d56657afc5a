# round 2 (3a): CTA-wide dense-tile queue (phase 2 per group) A/B + GPU tests
for lib in m dq0; do for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r3a.txt
done; done
python -m pytest tests -m gpu -q 2>&1 | tail -4 >> gpurun_out/r3a.txt
cat gpurun_out/r3a.txt
