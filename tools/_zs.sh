python -m pytest tests/test_gpu_parity_r2.py -x -q -k "zsolve" -s 2>&1 | grep -E "vs oracle|Error|assert|FAILED|passed|failed" | head -20
for r in 1 2; do for k in 0 1; do python tools/one_solve.py --cfg 4 --reps 10 --time --stages --tune 31=$k; done; done
for k in "31=1,30=2" "31=1,30=2,28=1" "31=1,30=1"; do python tools/one_solve.py --cfg 4 --reps 10 --time --stages --tune $k; done
