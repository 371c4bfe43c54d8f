NCU="ncu --clock-control none"
for cfg in "pi wlp 1000000 10000" "pi tlp 1000000 10000" "walk wlp 100000 1000" "walk tlp 100000 1000" "pi wlp 10000000 1000" "walk wlp 10000000 1000" "mm1 wlp 10000000 1000" "mm1 tlp 10000000 1000"; do
  set -- $cfg
  timeout 600 $NCU --set full --import-source on -k regex:"k_wlp|k_tlp" -s 1 -c 1 -o gpurun_out/r1i_$1_$2_$3 python tools/profile_driver.py $cfg --repeat 2 > gpurun_out/r1i_$1_$2_$3.log 2>&1
  echo "$cfg rc=$?"
done
timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1i_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > gpurun_out/r1i_bench_under_ncu.json 2>&1; echo launches rc=$?
