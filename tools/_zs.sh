python -m pytest tests/test_gpu_parity_r2.py -x -q -k "zsolve" 2>&1 | tail -1
for r in 1 2; do for k in "30=0" "30=1" "30=2" "30=1,28=1" "30=2,28=1"; do python tools/one_solve.py --cfg 4 --reps 10 --time --stages --tune $k; done; done
for k in "30=0" "30=1" "30=2" "30=1,28=1"; do python tools/one_solve.py --cfg 3 --reps 20 --time --stages --tune $k; done
