# round 2 (4f): CELLS component-major staged tile + two-shift entries + self pair in resolve() (c2)
# vs the halves build (h1); full GPU suite on c2
for lib in h1 c2; do
  for cfg in "3" "5" "5 --W 24" "4 --mode nearest" "6"; do
    echo "$lib cfg $cfg | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4f_ab.txt
  done
done
SPIN_LIB_PATH=abbuild/c2/libspin.so python -m pytest tests -m gpu -q -x 2>&1 | tail -5 >> gpurun_out/r4f_ab.txt
cat gpurun_out/r4f_ab.txt
