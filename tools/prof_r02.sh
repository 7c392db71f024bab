set -x
for k in 2 3; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast_k$k.csv python tools/ncu_cycle.py $k fast > gpurun_out/ncu_k$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_bottom -c 1 -s 2 -o gpurun_out/bottom_fast python tools/ncu_cycle.py 2 fast > gpurun_out/ncu_bottom.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pre -c 1 -s 1 -o gpurun_out/pre_fast python tools/ncu_cycle.py 2 fast > gpurun_out/ncu_pre.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_post -c 1 -s 4 -o gpurun_out/post_fast python tools/ncu_cycle.py 2 fast > gpurun_out/ncu_post.log 2>&1
ls -la gpurun_out
