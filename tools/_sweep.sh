for t in "" "29=0" "29=1" "14=2" "14=0" "3=4" "3=1" "2=3" "2=0" "13=0"; do
  echo "== tune $t"; timeout 120 python tools/one_solve.py --time --stages --reps 10 --tune "$t" 2>&1 | tail -3 | head -2
done
