export PYTHONPATH=.
set -x
# K10 variants at the measure() shapes (each after a plain run of the same command)
for cfg in ${CFGS:-"1000 10 2000 k10r_1000_p10" "10000 4 2000 k10mw_10000_p4"}; do
  set -- $cfg
  timeout 120 python tools/k10_once.py $1 $2 $3 > gpurun_out/plain_$4.txt 2>&1 && \
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:exec_free -c 1 -o gpurun_out/$4 python tools/k10_once.py $1 $2 $3 > gpurun_out/ncu_$4.log 2>&1
done
# K1c (variant 18) one 64-step pass at 2^28
[ -n "$K1C" ] && HEAT_SYNC_VARIANT=18 timeout 300 ncu --set full --import-source on --clock-control none -k regex:sync_cta -s 1 -c 1 -o gpurun_out/k1c_v18 python tools/probe_sync.py 268435456 128 > gpurun_out/ncu_k1c.log 2>&1
# K7 cfg1 and K9 cfg2 (the paper's configs)
[ -n "$K7" ] && timeout 300 ncu --set full --import-source on --clock-control none -k regex:sync_small -c 1 -o gpurun_out/k7_cfg1 python tools/k7_k9_once.py > gpurun_out/ncu_k7.log 2>&1
