# GPU session 61: unrolled 3x3 max-pool windows (group and padded pools)
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py tests/test_resnet_gpu.py -q -x > gpurun_out/t_61.log 2>&1; echo tests rc $?
for i in 1 2; do
  for mdl in googlenet resnet-50 inception-v3; do
    timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
    RALPB_LIB=abtest/base_mp.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/base /"
  done
done
tail -2 gpurun_out/t_61.log
