# GPU session 62: the per-step filter casts of branch groups / im2col layers batched into one launch
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py tests/test_resnet_gpu.py tests/test_step_gpu.py -q -x > gpurun_out/t_62.log 2>&1; echo tests rc $?
for i in 1 2; do
  for mdl in inception-v3 googlenet alexnet; do
    timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
    RALPB_LIB=abtest/base_cast.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/base /"
  done
done
tail -2 gpurun_out/t_62.log
