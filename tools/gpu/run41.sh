# GPU session 41: 'valid' stride-1 branch-group convs as cropped 'same' implicit convs
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_41.log 2>&1; echo tests rc $?
for i in 1 2; do for mdl in inception-v3 googlenet overfeat; do
  timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
  RALPB_MODULE_IMPLICIT=0 timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/im2col /"
done; done
tail -2 gpurun_out/t_41.log
