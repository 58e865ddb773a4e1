# GPU session 45: sibling groups of bias (non-batch-norm) 1x1 convs (GoogLeNet)
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_45.log 2>&1; echo tests rc $?
for i in 1 2; do
  timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null | sed "s/^/fuse /"
  RALPB_MODULE_FUSE=0 timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null | sed "s/^/nofuse /"
done
tail -2 gpurun_out/t_45.log
