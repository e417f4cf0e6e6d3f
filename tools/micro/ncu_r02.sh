# round-2 ncu evidence: one `ncu --set full` capture of the merge kernel per
# config (after warm-up launches), exported on the box as raw / source CSV
# pages (reports are large), then the launch list of the bench command
for c in C1 C2 C3 C4 C5 C2r C2t C4r X5; do
  timeout 600 ncu --set full --import-source on --clock-control none \
    -k regex:'merge_(pipe|small)_kernel' --launch-skip 3 -c 1 -o gpurun_out/r02_$c -f \
    python tools/run_config.py $c --reps 4 > gpurun_out/r02_ncu_$c.log 2>&1
  echo "$c rc=$?"
  ncu -i gpurun_out/r02_$c.ncu-rep --page raw --csv > gpurun_out/r02_ncu_raw_$c.csv 2>&1
  ncu -i gpurun_out/r02_$c.ncu-rep --page details --csv > gpurun_out/r02_ncu_details_$c.csv 2>&1
  [ "$c" = "C4" ] || [ "$c" = "C1" ] || rm -f gpurun_out/r02_$c.ncu-rep
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu \
  > gpurun_out/r02_ncu_bench.log 2>&1
echo "launch list rc=$?"
ls -la gpurun_out
