for t in "" "30=1" "30=2" "28=1" "28=1,30=1" "28=1,30=2" "26=4" "26=4,30=1"; do
  echo "== tune $t"; timeout 120 python tools/one_solve.py --time --stages --reps 10 --tune "$t" 2>&1 | tail -3 | head -2
done
