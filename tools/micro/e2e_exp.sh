tools/micro/e2e_model2 > gpurun_out/e2e_model_same.log 2>&1
for x in 0 1 2 3; do
  echo "exp $x: $(COMERGE_HOST_EXP=$x timeout 120 python tools/e2e_probe.py 2>&1 | tail -1)"
done > gpurun_out/e2e_exp.log
