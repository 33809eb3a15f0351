#!/bin/bash
# ncu captures summarised on the box (the .ncu-rep files are too large to bring back together)
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu > gpurun_out/b_ncu.log 2>&1
for k in sweep_kernel post_gradB_blk_kernel cut_kernel post_prep_kernel post_pos_kernel; do
  skip=0; [ "$k" != sweep_kernel ] && skip=20
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/ncu_$k -f python tools/one_posterior.py c4 full > gpurun_out/ncu_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$k.ncu-rep gpurun_out/r02_ncu_${k}_summary.txt $( [ $k = sweep_kernel ] && echo --traffic-json gpurun_out/r02_sweep_traffic.json ) > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/ncu_$k.ncu-rep 0 30 > gpurun_out/r02_ncu_${k}_lines.txt 2>&1
done
cp /tmp/ncu_sweep_kernel.ncu-rep gpurun_out/r02_ncu_sweep.ncu-rep
ls -la gpurun_out/
