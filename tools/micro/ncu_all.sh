# one `ncu --set full` capture of the merge kernel per config (after warm-up launches)
for c in C1 C2 C3 C4 C5; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_pipe_kernel \
    --launch-skip 3 -c 1 -o gpurun_out/r01_$c -f python tools/run_config.py $c --reps 4 > gpurun_out/r01_ncu_$c.log 2>&1
  echo "$c rc=$?"
done
