mkdir -p gpurun_out/nc
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc -s 1 -c 1 \
  -o gpurun_out/nc/conv96 -f python tools/ncu_conv_one.py 21 720 1280 96 96 > gpurun_out/nc/ncu96.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/nc/ncu96.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc -s 1 -c 1 \
  -o gpurun_out/nc/conv192 -f python tools/ncu_conv_one.py 21 360 640 192 192 > gpurun_out/nc/ncu192.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/nc/ncu192.log
