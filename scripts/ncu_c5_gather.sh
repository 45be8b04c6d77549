timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gather_u8_pieces" -s 20 -c 1 -o gpurun_out/ncu_gu8 python scripts/dp1_c5_timing.py > gpurun_out/ncu_gu8.log 2>&1
echo rc=$?
