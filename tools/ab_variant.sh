#!/bin/bash
# Same-box check of a variant build (tools/build_variant.sh NAME ...) against the
# default library: bitwise fingerprints of cfg1-4 solves in both workspace layouts
# (tools/bits.py), alternating timed runs (tools/ab.py) and per-launch stage times.
#   bash tools/ab_variant.sh NAME        (writes gpurun_out/bits_*.txt, ab_NAME*.txt)
A=paper_1912_03565_b200/_lib/libhelmfft_b200.so
B=paper_1912_03565_b200/_lib/libhelmfft_b200_${1:-addr}.so
HFB_LIBRARY=$A timeout 200 python tools/bits.py 1 2 3:63 3:255 3 4 > gpurun_out/bits_A.txt 2>&1
HFB_LIBRARY=$B timeout 200 python tools/bits.py 1 2 3:63 3:255 3 4 > gpurun_out/bits_B.txt 2>&1
diff gpurun_out/bits_A.txt gpurun_out/bits_B.txt && echo BITS_EQUAL
cat gpurun_out/bits_B.txt
timeout 400 python tools/ab.py --rounds 3 $A $B > gpurun_out/ab_$1.txt 2>&1; cat gpurun_out/ab_$1.txt
for L in $A $B; do HFB_LIBRARY=$L timeout 120 python tools/one_solve.py --time --stages --reps 10 2>&1 | tail -3; done | tee gpurun_out/ab_$1_stages.txt
