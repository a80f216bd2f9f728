#!/bin/bash
# bench + ncu evidence for profiles/ (one GPU). Usage: bash tools/profile_round.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p2g|k_g2p" -s 4 -c 2 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
