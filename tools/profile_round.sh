#!/bin/bash
# bench + ncu evidence for profiles/ (one GPU). Usage: bash tools/profile_round.sh <tag> [kernel-regex]
# Each ncu pass runs only after the same command exited 0 without ncu.
TAG=${1:-r02}
KRE=${2:-"k_p2g|k_g2p|k_grid|k_inc_block"}
mkdir -p gpurun_out
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-workloads --adj-steps 0"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 12 -c 4 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
