# A/B timing of the CELLS configs for the default library or SPIN_LIB_PATH builds
for lib in ${LIBS:-paper_1811_00901_b200/libspin.so}; do
  for c in ${CFGS:-3 5}; do
    SPIN_LIB_PATH=$lib python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['workload'], d['config']['mode'], round(d['ms_per_step'],2), 'G', d['config']['G'])"
  done
done
