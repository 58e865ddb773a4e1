# GPU session 60: bias convs' relu-grad + pad + column sum in one pass
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_60.log 2>&1; echo tests rc $?
for i in 1 2; do
  for mdl in googlenet inception-v3 overfeat; do
    timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
    RALPB_LIB=abtest/base_rg.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/base /"
  done
done
tail -2 gpurun_out/t_60.log
