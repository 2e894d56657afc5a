# A/B timing of library builds (LIBS, loaded through SPIN_LIB_PATH) over a list of bench
# argument sets (ARGS, ';'-separated); one line per (lib, args)
IFS=';' read -ra SETS <<< "${ARGS:---config 2 --mode bilinear;--config 2 --mode nearest;--config 6;--config 3;--config 5}"
for lib in ${LIBS:-paper_1811_00901_b200/libspin.so}; do
  for a in "${SETS[@]}"; do
    SPIN_LIB_PATH=$lib python bench.py $a --no-cpu-baseline --no-e2e --steps ${STEPS:-5} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$a', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
  done
done
