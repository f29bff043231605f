timeout 300 python tools/latency_probe.py 100 200000 100 40 > gpurun_out/lat.log 2>&1
for k in fused incremental; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 20 --launch-count 1 -o gpurun_out/r02_lat_$k -f python tools/latency_probe.py 100 200000 100 25 $k >> gpurun_out/lat.log 2>&1
done
