# kernel time vs the static share of the tiles (the rest is the dynamic tail)
for c in ${CFGS:-C2 C4 C5 X1}; do for sp in ${PCTS:-60 65 70 75 80}; do
  timeout 120 python tools/ab.py $c 0 --static-pct $sp --rounds 2 | sed "s/flags=0/static=$sp/"
done; done
