# GPU session 26: same-box A/B sweep of the runtime knobs on the headline step (bench --quick)
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --quick > gpurun_out/ab_$tag.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$tag.json').readline()); print('$tag', round(d['ms_per_step'],3), round(d['value']), d['clocks']['sm_mhz'])"; }
run base0 X=0
run nb4 RALPB_NB=4
run nb6 RALPB_NB=6
run acc1 RALPB_ACC_BUFS=1
run pdl0 RALPB_PDL=0
run fcov0 RALPB_FC_OVERLAP=0
run poolidx RALPB_POOL_IDX=1
run base1 X=1
run fwdpair0 RALPB_FWD_PAIR=0
run graph0 RALPB_GRAPH=0
run base2 X=2
