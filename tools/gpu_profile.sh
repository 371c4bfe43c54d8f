# ncu captures of the replication kernels (one launch each), the bench launch list, and a
# cross-check of the instrumented memory counters against ncu's global ld/st counts.
# usage: bash tools/gpu_profile.sh TAG
TAG=${1:-r1}
NCU="ncu --clock-control none"
timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > /dev/null 2>&1
for cfg in "pi wlp 1000000 10000" "pi tlp 1000000 10000" "walk wlp 100000 1000" "walk tlp 100000 1000" "mm1 tlp 1000000 1000" "mm1 wlp 1000000 1000" "pi wlp 10000000 1000" "walk wlp 10000000 1000"; do
  set -- $cfg
  timeout 600 $NCU --set full --import-source on -k regex:"k_wlp|k_tlp" -s 1 -c 1 -o gpurun_out/${TAG}_$1_$2_$3 python tools/profile_driver.py $cfg --repeat 2 > /dev/null 2>&1
  echo "$cfg rc=$?"
done
# counters vs ncu (instrumented kernels): global load/store warp-instructions
for cfg in "walk tlp 100000 1000" "walk wlp 100000 1000" "mm1 tlp 100000 1000" "mm1 wlp 100000 1000"; do
  set -- $cfg
  timeout 300 $NCU --metrics smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_st.sum -k regex:"k_wlp|k_tlp" -s 1 -c 1 python tools/profile_driver.py $cfg --repeat 2 --counters > gpurun_out/${TAG}_counters_$1_$2.txt 2>&1
  echo "counters $cfg rc=$?"
done
