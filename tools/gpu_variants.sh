# ncu evidence on the cfg 4 grid: resident-q forward and backward (dev tool)
P="python tools/profile_step.py --config 4 --shots 4 --nt 60 --reps 1"
$P > /dev/null 2>&1; echo plain=$?
ncu --set full --clock-control none -k regex:fwd_qres -s 20 -c 1 -o gpurun_out/prof_qres_cfg4 $P > gpurun_out/ncu_qres.log 2>&1; echo q=$?
ncu --set full --clock-control none -k regex:bwd_step -s 20 -c 1 -o gpurun_out/prof_bwd_cfg4 $P > gpurun_out/ncu_bwd4.log 2>&1; echo b=$?
