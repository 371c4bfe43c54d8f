NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:"k_wlp_mm1" -s 1 -c 1 -o gpurun_out/prof_mm1_wlp_v2 python tools/profile_driver.py mm1 wlp 1000000 1000 --repeat 2 > gpurun_out/prof_mm1_wlp_v2.log 2>&1
echo rc=$?
