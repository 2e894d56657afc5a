# round 2 (5f): C4 NEAREST on the final build (two rows per dense-walk step): stage times and ncu --set full
for sk in 0 1 2; do
  echo "cfg 4 --mode nearest skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config 4 --mode nearest 2>&1 | tail -1)" >> gpurun_out/r5f_stages.txt
done
ncu -k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on -o gpurun_out/r5f_c4nearest python tools/one_call.py --config 4 --mode nearest > gpurun_out/r5f_ncu.log 2>&1
cat gpurun_out/r5f_stages.txt
