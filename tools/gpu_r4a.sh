# round 2 (4a): re-entry check of HEAD on a fresh box: GPU tests, default bench, CELLS timings
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r4a_tests.txt
python bench.py > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
CFGS="3 5" bash tools/ab_cells.sh > gpurun_out/r4a_cells.txt 2>&1
python tools/one_call.py --config 5 --W 24 >> gpurun_out/r4a_cells.txt 2>&1
tail -3 gpurun_out/r4a_tests.txt; tail -c 600 gpurun_out/r4a_bench.json; cat gpurun_out/r4a_cells.txt
