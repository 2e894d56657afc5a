# round 2 (4j): evidence of the final round-2 build (pinned dense-walk address, CELLS accept-path
# trims, self pair in resolve()): GPU suite, default bench + reference arm, stage table per config
# (measurement build), ncu launch list of the bench and --set full of one launch per config
python -m pytest tests -m gpu -q --durations=12 2>&1 | tail -22 > gpurun_out/r4j_tests.txt
python bench.py > gpurun_out/r4j_bench.json 2> gpurun_out/r4j_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r4j_ref.json 2> gpurun_out/r4j_ref.err
python bench.py --config 2 --no-cpu-baseline --no-dls > gpurun_out/r4j_bench_c2.json 2> gpurun_out/r4j_bench_c2.err
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6" "3" "5" "5 --W 24"; do
  for sk in 0 1 2; do
    echo "cfg $cfg skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4j_stages.txt
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4j_launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dls > gpurun_out/r4j_ncu_launch.log 2>&1
K="-k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on"
for spec in "4:" "4:--mode nearest" "2:" "3:" "5:" "5:--W 24"; do
  c=${spec%%:*}; extra=${spec#*:}; tag=c${c}$(echo "$extra" | tr -d ' -' | sed 's/mode//;s/W/w/')
  ncu $K -o gpurun_out/r4j_$tag python tools/one_call.py --config $c $extra > gpurun_out/r4j_ncu_$tag.log 2>&1
done
tail -3 gpurun_out/r4j_tests.txt; tail -c 300 gpurun_out/r4j_bench.json; cat gpurun_out/r4j_stages.txt; ls -la gpurun_out | grep r4j
