python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -c 600 gpurun_out/bench2.json
