# Bitsliced walk kernels (all three), ncu --set full, summarised on the box.
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:"k_wlp_walk_bs_lanes" -s 1 -c 1 -o gpurun_out/r1l_walk_wlpbslanes_100000 python tools/profile_driver.py walk wlp 100000 1000 --repeat 2 > gpurun_out/r1l_a.log 2>&1; echo a rc=$?
timeout 600 $NCU --set full --import-source on -k regex:"k_wlp_walk_bs_pipe" -s 1 -c 1 -o gpurun_out/r1l_walk_wlpbspipe_10000000 python tools/profile_driver.py walk wlp 10000000 1000 --repeat 2 > gpurun_out/r1l_b.log 2>&1; echo b rc=$?
timeout 600 $NCU --set full --import-source on -k regex:"k_tlp_walk_bs" -s 1 -c 1 -o gpurun_out/r1l_walk_tlpbs_10000000 python tools/profile_driver.py walk tlp 10000000 1000 --repeat 2 --tlp-variant 2 > gpurun_out/r1l_c.log 2>&1; echo c rc=$?
timeout 600 $NCU --set full --import-source on -k regex:"k_tlp_walk_bs" -s 1 -c 1 -o gpurun_out/r1l_walk_tlpbs_100000 python tools/profile_driver.py walk tlp 100000 1000 --repeat 2 --tlp-variant 2 > gpurun_out/r1l_d.log 2>&1; echo d rc=$?
python tools/ncu_summary.py gpurun_out/round1_ncu_v8 gpurun_out/r1l_*.ncu-rep; echo summary rc=$?
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
python tools/ncu_lines.py gpurun_out/r1l_walk_tlpbs_10000000.ncu-rep 30 > gpurun_out/round1_walk_tlp_bitsliced_source_lines.txt
python tools/ncu_lines.py gpurun_out/r1l_walk_wlpbslanes_100000.ncu-rep 30 > gpurun_out/round1_walk_wlp_bitsliced_lanes_source_lines.txt
rm -f gpurun_out/r1l_*.ncu-rep
