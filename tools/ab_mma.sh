# A/B of the BRUTE sphere filter: tensor cores (default) vs packed fp32 (SPIN_NO_MMA=1),
# whole kernel and with the accept path / compaction switched off (SPIN_DEBUG_SKIP)
for skip in ${SKIPS:-0 1 2}; do
for env in "" "SPIN_NO_MMA=1"; do
  for c in ${CONFIGS:-"--config 2 --mode bilinear" "--config 2 --mode nearest" "--config 6"}; do
    env SPIN_DEBUG_SKIP=$skip $env python bench.py $c --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$skip', '$env', '$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['pairs'])"
  done
done
done
