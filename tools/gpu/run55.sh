# GPU session 55: batch-norm reductions finished by their last block (no memset / finish / params launches)
set -x
timeout 1500 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_55.log 2>&1; echo tests rc $?
for i in 1 2; do
  for lib in new base; do
    for mdl in inception-v3 resnet-50 googlenet; do
      if [ $lib = base ]; then
        RALPB_LIB=abtest/base_bn.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/$lib /"
      else
        timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/$lib /"
      fi
    done
  done
done
tail -2 gpurun_out/t_55.log
