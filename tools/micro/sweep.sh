timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python tools/ab.py C4 0,512 --rounds 2
for c in C1 C2 C3 C5; do timeout 300 python tools/ab.py $c 0 --rounds 2; done
