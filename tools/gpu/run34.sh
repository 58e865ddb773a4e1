# GPU session 34: same-box A/B of build variants (first-conv producer warpgroups)
run() { tag=$1; lib=$2; RALPB_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --quick > gpurun_out/ab34_$tag.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/ab34_$tag.json').readline()); print('$tag', round(d['ms_per_step'],3), round(d['value']), d['clocks']['sm_mhz'], d['roofline']['by_kind'].get('first_conv_fwd'))"; }
B=paper_1901_05803_b200/libralpb200.so
run base_a $B; run g4_a abtest/first_g4.so; run g2_a abtest/first_g2.so
run base_b $B; run g4_b abtest/first_g4.so; run g2_b abtest/first_g2.so
