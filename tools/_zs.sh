python -m pytest tests/test_gpu_parity_r2.py -x -q -k "zsolve" 2>&1 | tail -1
for r in 1 2; do for k in 0 1; do python tools/one_solve.py --cfg 4 --reps 10 --time --stages --tune 28=$k; done; done
for k in 0 1; do python tools/one_solve.py --cfg 3 --reps 20 --time --stages --tune 28=$k; done
