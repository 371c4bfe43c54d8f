# GPU check after the mm1 rework: tests, bench, ncu on mm1 kernels
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench_rc=$?; tail -3 gpurun_out/bench2.err
NCU="ncu --clock-control none"
for cfg in "mm1 tlp 1000000 1000" "mm1 wlp 1000000 1000" "pi wlp 1000000 10000"; do
  set -- $cfg
  timeout 600 $NCU --set full --import-source on -k regex:"k_wlp|k_tlp" -s 1 -c 1 -o gpurun_out/prof2_$1_$2 python tools/profile_driver.py $cfg --repeat 2 > gpurun_out/prof2_$1_$2.log 2>&1
  echo "$cfg rc=$?"
done
