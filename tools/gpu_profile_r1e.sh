set -x
NCU="ncu --clock-control none"
for cfg in "mm1 wlp 1000000 1000" "mm1 tlp 1000000 1000" "pi wlp 1000000 10000" "walk wlp 10000000 1000"; do
  set -- $cfg
  timeout 600 $NCU --set full --import-source on -k regex:"k_wlp|k_tlp" -s 1 -c 1 -o gpurun_out/r1e_$1_$2_$3 python tools/profile_driver.py $cfg --repeat 2 > gpurun_out/r1e_$1_$2_$3.log 2>&1
  echo "$cfg rc=$?"
done
timeout 600 $NCU --set full --import-source on -k regex:"k_wlp_mm1" -s 1 -c 1 -o gpurun_out/r1e_mm1_wlp_rho95 python tools/profile_driver.py mm1 wlp 1000000 1000 --lambda 0.95 --repeat 2 > gpurun_out/r1e_mm1_rho95.log 2>&1; echo rho95 rc=$?
timeout 600 $NCU --set full --import-source on -k regex:"k_ir" -s 0 -c 1 -o gpurun_out/r1e_ir_walk_tlp python tools/profile_driver.py walk tlp 20000 1000 --ir --repeat 1 > gpurun_out/r1e_ir.log 2>&1; echo ir rc=$?
timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1e_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > gpurun_out/r1e_bench_under_ncu.json 2>&1; echo launches rc=$?
ls -la gpurun_out | tail -20
