# GPU session 66: four producer warps (416-thread GEMM CTAs) vs the 384-thread three-producer build
set -x
for i in 1 2; do
  for lib in new base; do
    for mdl in inception-v3 resnet-50 googlenet; do
      if [ $lib = base ]; then RALPB_LIB=abtest/base_p3.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/$lib /";
      else timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/$lib /"; fi
    done
    if [ $lib = base ]; then RALPB_LIB=abtest/base_p3.so timeout 600 python bench.py --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib vgg16b', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])";
    else timeout 600 python bench.py --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib vgg16b', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; fi
  done
done
