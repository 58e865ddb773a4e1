# GPU session 70: relu-grad + bias-sum pass two items in flight per thread
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_70.log 2>&1; echo tests rc $?
for i in 1 2; do
  for mdl in googlenet overfeat; do
    timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
    RALPB_LIB=abtest/base_u2.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/base /"
  done
done
tail -2 gpurun_out/t_70.log
