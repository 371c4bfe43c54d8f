set -x
./tools/microbench > gpurun_out/microbench.txt 2>&1
cat gpurun_out/microbench.txt
NCU="ncu --clock-control none"
timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > gpurun_out/bench_under_ncu.json 2>&1
for cfg in "pi wlp 1000000 10000" "pi tlp 1000000 10000" "walk wlp 100000 1000" "walk tlp 100000 1000" "mm1 tlp 1000000 1000" "mm1 wlp 1000000 1000"; do
  set -- $cfg
  timeout 600 $NCU --set full --import-source on -k regex:"k_wlp|k_tlp" -s 1 -c 1 -o gpurun_out/prof_$1_$2 python tools/profile_driver.py $cfg --repeat 2 > gpurun_out/prof_$1_$2.log 2>&1
  echo "$cfg rc=$?"
done
ls -la gpurun_out
