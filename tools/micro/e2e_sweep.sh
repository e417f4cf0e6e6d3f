# e2e (host pinned buffers, C2 shape) vs host pipeline chunk count, with per-chunk traces
for c in ${CHUNKS:-6 8 12 16}; do
  echo "chunks $c: $(COMERGE_HOST_CHUNKS=$c COMERGE_HOST_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/e2e_c$c.trace | tail -1)"
done > gpurun_out/e2e_sweep.log
