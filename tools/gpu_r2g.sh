# round 2 (g): stage breakdown of C4 BILINEAR with / without dense tiles, then ncu of the dense build
for dm in 0 8; do for sk in 0 1 2; do
  echo "dense_min $dm skip $sk: $(SPIN_DENSE_MIN=$dm SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so python tools/one_call.py --config 4 2>&1 | tail -1)" >> gpurun_out/r2g.txt
done; done
cat gpurun_out/r2g.txt
ncu -k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on -o gpurun_out/r2g_c4 python tools/one_call.py --config 4 > gpurun_out/r2g_ncu.log 2>&1
tail -3 gpurun_out/r2g_ncu.log
