for c in C2 X1 C4 C3; do
 for f in 0 1 0 1; do
  echo "$c flags=$f $(timeout 120 python tools/run_config.py $c --reps 5 --flags $f --trace 2>&1 | grep -E 'rep 4|first tile|startup' | tr '\n' ' ')"
 done
done
