#!/bin/bash
# Final round-2 ncu captures (run on the GPU box, one GPU): launch lists of
# eager n=12 cycles (kappa 2, 3; FMA build) and --set full reports of the
# level-1 pre pass, the level-1 post pass and the bottom kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for k in 2 3; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast_k$k.csv \
      python tools/ncu_cycle.py $k fast > gpurun_out/ncu_k$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_bottom -c 1 -s 2 -f -o gpurun_out/bottom_fast \
    python tools/ncu_cycle.py 3 fast > gpurun_out/ncu_bottom.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pre -c 1 -s 0 -f -o gpurun_out/pre1_fast \
    python tools/ncu_cycle.py 3 fast > gpurun_out/ncu_pre.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_post -c 1 -s 6 -f -o gpurun_out/post1_fast \
    python tools/ncu_cycle.py 3 fast > gpurun_out/ncu_post.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
