# stage breakdown (SPIN_DEBUG_SKIP: 1 = no accept path, 2 = no compaction either) per config
for cfg in "3" "5" "5 --W 24" "2" "4" "4 --mode nearest"; do
  for skip in 0 1 2; do
    SPIN_DEBUG_SKIP=$skip SPIN_LIB_PATH=abbuild/m0/libspin.so timeout 300 python bench.py --config $cfg --steps 5 --no-cpu-baseline --no-e2e --no-dls > /tmp/o.json 2>/dev/null
    python -c "
import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('cfg $cfg skip $skip', round(d['roofline']['kernel_ms'],2), d['config']['G'], d['pairs']['visited'], d['pairs']['candidate'], d['pairs']['accepted'])"
  done
done
