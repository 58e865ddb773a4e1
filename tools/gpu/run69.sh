# GPU session 69: ResNet-50 blocks' per-step operand copies through the batched cast / prep launches
set -x
timeout 1500 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_69.log 2>&1; echo tests rc $?
for i in 1 2; do
  for mdl in resnet-50; do
    timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
    RALPB_LIB=abtest/base_bp.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/base /"
  done
done
tail -2 gpurun_out/t_69.log
