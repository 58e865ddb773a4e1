# GPU session 54: VGG-16 A/B of the K-major third producer (bench --quick lines)
set -x
for i in 1 2 3; do
  for k in 2 3; do
    RALPB_GEMM_PRODUCERS_K=$k timeout 600 python bench.py --quick 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('k$k', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
