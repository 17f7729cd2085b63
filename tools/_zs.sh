python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -c 300 gpurun_out/bench3.json
for c in 1 2 3; do python tools/one_solve.py --cfg $c --reps 20 --time --stages; done
