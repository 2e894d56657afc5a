# round 2 (p): dense loop variants in ONE call (row list 2 rows / 1 row / bit scan; defer on/off)
for rep in 1 2; do for lib in m dr1 dl0 dl0nd; do for cfg in "4" "4 --mode nearest"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2p.txt
done; done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> gpurun_out/r2p.txt
cat gpurun_out/r2p.txt
