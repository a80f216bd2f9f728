#!/bin/bash
# fwd+adjoint evidence for profiles/ (one GPU): device-timed checkpointed backprop at C4 f64,
# the launch list of one backprop call and a full ncu capture of the four adjoint kernels inside it.
# Usage: bash tools/profile_adj.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python tools/bench_adjoint.py C4 10 2"
$CMD > gpurun_out/${TAG}_adj_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -s 200 -c 300 --csv \
    --log-file gpurun_out/${TAG}_adj_launches.csv $CMD > gpurun_out/${TAG}_adj_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_adj" -s 16 -c 4 \
    -o gpurun_out/${TAG}_adj_full $CMD > gpurun_out/${TAG}_adj_ncu_full.log 2>&1
echo "ncu rc=$?"
