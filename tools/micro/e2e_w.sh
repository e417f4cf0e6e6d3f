# e2e (C2 shape) for explicit chunk weight lists
for wl in "1,1,1,1,1,1,1,1" "0.5,1,1,1,1,1,1,1,0.5" "0.25,0.25,0.5,1,1,1,1,1,1,0.5,0.25,0.25" "0.5,0.5,1,1,1,1,1,1,1,0.5,0.5" "0.75,1,1,1,1,1,1,1,0.25" "1,1,1,1,1,1,1,0.5,0.5" "0.5,0.5,1,1,1,1,1,1,1"; do
  echo "weights $wl: $(COMERGE_HOST_WEIGHTS=$wl COMERGE_HOST_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/e2e_w_$wl.trace | tail -1)"
done > gpurun_out/e2e_w.log
