# e2e (host pinned buffers, C2 shape) vs host pipeline chunking (parts x end ramp), per-chunk traces
for c in ${CHUNKS:-6 8 12}; do for r in ${RAMPS:-0 1 2 3}; do
  echo "parts $c ramp $r: $(COMERGE_HOST_CHUNKS=$c COMERGE_HOST_RAMP=$r COMERGE_HOST_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/e2e_c${c}_r$r.trace | tail -1)"
done; done > gpurun_out/e2e_sweep.log
