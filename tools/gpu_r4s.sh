# round 2 (4s): last check after the measurement-knob commit: smoke, GPU suite, default bench
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1 > gpurun_out/r4s_check.txt
python -m pytest tests -m gpu -q 2>&1 | tail -1 >> gpurun_out/r4s_check.txt
python bench.py 2> gpurun_out/r4s_bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])" >> gpurun_out/r4s_check.txt
cat gpurun_out/r4s_check.txt
