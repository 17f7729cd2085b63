python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -c 200 gpurun_out/bench4.json
