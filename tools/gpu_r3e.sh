# round 2 (3e): evidence of the fragment-tile build (same steps as gpu_r2z.sh)
# stage breakdown per config (measurement build), ncu launch list of the bench and --set full of C4
python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r3e_tests.txt
python bench.py > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r3e_ref.json 2> gpurun_out/r3e_ref.err
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6" "3" "5" "5 --W 24"; do
  for sk in 0 1 2; do
    echo "cfg $cfg skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r3e_stages.txt
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3e_launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dls > gpurun_out/r3e_ncu_launch.log 2>&1
ncu -k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on -o gpurun_out/r3e_c4 python tools/one_call.py --config 4 > gpurun_out/r3e_ncu_c4.log 2>&1
ncu -k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on -o gpurun_out/r3e_c4n python tools/one_call.py --config 4 --mode nearest > gpurun_out/r3e_ncu_c4n.log 2>&1
ncu -k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on -o gpurun_out/r3e_c2 python tools/one_call.py --config 2 > gpurun_out/r3e_ncu_c2.log 2>&1
tail -3 gpurun_out/r3e_tests.txt; tail -c 400 gpurun_out/r3e_bench.json; cat gpurun_out/r3e_stages.txt
