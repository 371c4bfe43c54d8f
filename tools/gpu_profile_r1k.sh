# Bitsliced walk kernels: ncu --set full (config 4 and 3), summarised on the box.
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:"k_wlp_walk_bs_pipe" -s 1 -c 1 -o gpurun_out/r1k_walk_wlpbs_10000000 python tools/profile_driver.py walk wlp 10000000 1000 --repeat 2 > gpurun_out/r1k_a.log 2>&1; echo a rc=$?
timeout 600 $NCU --set full --import-source on -k regex:"k_tlp_walk_bs" -s 1 -c 1 -o gpurun_out/r1k_walk_tlpbs_10000000 python tools/profile_driver.py walk tlp 10000000 1000 --repeat 2 --tlp-variant 2 > gpurun_out/r1k_b.log 2>&1; echo b rc=$?
timeout 600 $NCU --set full --import-source on -k regex:"k_tlp_walk_bs" -s 1 -c 1 -o gpurun_out/r1k_walk_tlpbs_100000 python tools/profile_driver.py walk tlp 100000 1000 --repeat 2 --tlp-variant 2 > gpurun_out/r1k_c.log 2>&1; echo c rc=$?
python tools/ncu_summary.py gpurun_out/round1_ncu_v8 gpurun_out/r1k_*.ncu-rep; echo summary rc=$?
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
python tools/ncu_lines.py gpurun_out/r1k_walk_tlpbs_10000000.ncu-rep 30 > gpurun_out/round1_walk_tlp_bitsliced_source_lines.txt
rm -f gpurun_out/r1k_*.ncu-rep
