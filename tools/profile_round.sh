#!/bin/bash
# Round-end evidence for profiles/ (run on the GPU box after `python bench.py` exited 0 without ncu):
#   1. DRAM bytes + duration of every walk launch of 2 projections (warmup 1 + step 1)
#   2. the launch list (all kernels, ~1 projection) for the kernel shares
#   3. one mid-projection walk launch under --set full (instructions per iteration, issue, stalls)
#   4. one busy wave of the other kernels under --set full
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ktime"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:wave_walk --csv --log-file gpurun_out/walk_dram.csv $B > gpurun_out/ncu_dram.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
XSCAT_WAVE_PIPES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:wave_walk -s 12 -c 1 -o gpurun_out/walk_full -f $B > gpurun_out/ncu_walk.log 2>&1
XSCAT_WAVE_PIPES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"wave_(setup|score|event|admit)" -s 40 -c 4 -o gpurun_out/nonwalk_full -f $B > gpurun_out/ncu_nonwalk.log 2>&1
echo done
