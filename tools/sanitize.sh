#!/bin/bash
# compute-sanitizer evidence for profiles/ (one GPU): racecheck and synccheck of the shared-memory
# kernels (P2G column march, the G2P-transpose scatter, the incremental sort), memcheck of all.
mkdir -p gpurun_out
D="python tools/sanitize_driver.py"
$D > gpurun_out/san_plain.log 2>&1 || { echo "driver failed"; exit 1; }
for tool in racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name regex:"k_p2g|k_adj_scatter|k_inc_|k_g2p|k_adj_g2pT" \
    $D > gpurun_out/san_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.txt
  tail -3 gpurun_out/san_${tool}.log >> gpurun_out/san_summary.txt
done
timeout 1500 compute-sanitizer --tool memcheck $D > gpurun_out/san_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/san_summary.txt
tail -3 gpurun_out/san_memcheck.log >> gpurun_out/san_summary.txt
