# e2e (C2 shape) per host-pipeline chunk count
for c in ${CHUNKS:-7 8 9 10}; do
  echo "chunks $c: $(COMERGE_HOST_CHUNKS=$c timeout 120 python tools/e2e_probe.py 2>&1 | tail -1)"
done
