A=paper_1912_03565_b200/_lib/libhelmfft_b200_old.so
B=paper_1912_03565_b200/_lib/libhelmfft_b200.so
C=paper_1912_03565_b200/_lib/libhelmfft_b200_noxor.so
for r in 1 2; do for L in $A $B $C; do echo "== $L cfg5"; HFB_LIBRARY=$L timeout 200 python tools/one_solve.py --cfg 5 --time --stages --reps 3 2>&1 | tail -3 | head -2; done; done
for t in "29=0" "14=0" "13=0"; do echo "== new cfg5 tune $t"; HFB_LIBRARY=$B timeout 200 python tools/one_solve.py --cfg 5 --time --stages --reps 3 --tune $t 2>&1 | tail -3 | head -2; done
