timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in C2 X1 C4 C3 C5; do
 for sp in 0 60 65 70 80; do
  echo "$c sp=$sp $(timeout 120 python tools/run_config.py $c --reps 6 --static-pct $sp 2>&1 | grep -E 'rep 5' | tr '\n' ' ')"
 done
done
