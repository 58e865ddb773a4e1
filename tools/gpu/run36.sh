# GPU session 36: same-box A/B of the residual-add epilogue (RALPB_RES_EPI=0 vs default)
for i in 1 2; do
for v in 1 0; do
  for mdl in resnet-50 inception-v3 googlenet; do
    RALPB_RES_EPI=$v timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/res_epi=$v /"
  done
done
done
RALPB_RES_EPI=0 timeout 900 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py -q -x -k "teacher" 2>&1 | tail -1
