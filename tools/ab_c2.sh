# A/B timing of C2 (and optionally C4) for the default library or SPIN_LIB_PATH builds
for lib in ${LIBS:-paper_1811_00901_b200/libspin.so}; do
  for m in bilinear nearest; do
    for sup in auto first; do
      SPIN_LIB_PATH=$lib python bench.py --config 2 --mode $m --no-cpu-baseline --no-e2e --steps 10 --support $sup 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['mode'], '$sup', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
    done
  done
done
