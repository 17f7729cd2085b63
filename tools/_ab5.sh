A=paper_1912_03565_b200/_lib/libhelmfft_b200_old.so
B=paper_1912_03565_b200/_lib/libhelmfft_b200.so
for r in 1 2; do for L in $A $B; do echo "== $L cfg5"; HFB_LIBRARY=$L timeout 200 python tools/one_solve.py --cfg 5 --time --stages --reps 3 2>&1 | tail -3 | head -2; done; done
for L in $A $B; do echo "== $L cfg3"; HFB_LIBRARY=$L timeout 100 python tools/one_solve.py --cfg 3 --time --stages --reps 20 2>&1 | tail -3 | head -2; done
for L in $A $B; do echo "== $L cfg2"; HFB_LIBRARY=$L timeout 100 python tools/one_solve.py --cfg 2 --time --stages --reps 50 2>&1 | tail -3 | head -2; done
for L in $A $B; do echo "== $L complex"; HFB_LIBRARY=$L timeout 200 python tools/one_solve_z.py 2>&1 | tail -3; done
