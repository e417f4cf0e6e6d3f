timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in C2 X1 C4 C5 C3 C1; do
 for sp in 0 70 60; do
  echo "$c sp=$sp $(timeout 120 python tools/run_config.py $c --reps 5 --static-pct $sp --trace 2>&1 | grep -E 'rep 4|first tile|  end ' | tr '\n' ' ')"
 done
done
