# round-2 profiles: plain run, then ncu --set full of the second spin_persistent launch,
# and launch lists of the bench default (C4) and C5
set -x
K="-k regex:spin_persistent -s 1 -c 1 --set full --clock-control none --import-source on"
for spec in "4:" "4:--mode nearest" "2:" "3:" "5:" "5:--W 24"; do
  c=${spec%%:*}; extra=${spec#*:}; tag=c${c}$(echo "$extra" | tr -d ' -' | sed 's/mode//;s/W/w/')
  python tools/one_call.py --config $c $extra > gpurun_out/r2e_plain_$tag.log 2>&1 && \
  ncu $K -o gpurun_out/r2e_$tag python tools/one_call.py --config $c $extra > gpurun_out/r2e_ncu_$tag.log 2>&1
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dls > gpurun_out/r2e_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dls > gpurun_out/r2e_ncu_launch.log 2>&1
ls -la gpurun_out/ | grep r2e
