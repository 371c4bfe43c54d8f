# Round-1 final captures: ncu --set full per kernel/config, summarised ON the box (the
# .ncu-rep files together exceed gpurun's 64 MiB return limit), the launch list of the
# bench command, and a plain bench run.
NCU="ncu --clock-control none"
for cfg in "pi wlp 1000000 10000" "pi tlp 1000000 10000" "walk wlp 100000 1000" "walk tlp 100000 1000" "pi wlp 10000000 1000" "walk wlp 10000000 1000" "mm1 wlp 10000000 1000" "mm1 tlp 10000000 1000"; do
  set -- $cfg
  timeout 600 $NCU --set full --import-source on -k regex:"k_wlp|k_tlp" -s 1 -c 1 -o gpurun_out/r1j_$1_$2_$3 python tools/profile_driver.py $cfg --repeat 2 > gpurun_out/r1j_$1_$2_$3.log 2>&1
  echo "$cfg rc=$?"
done
python tools/ncu_summary.py gpurun_out/round1_ncu_v7 gpurun_out/r1j_*.ncu-rep; echo summary rc=$?
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
python tools/ncu_lines.py gpurun_out/r1j_pi_wlp_1000000.ncu-rep 40 > gpurun_out/round1_pi_wlp_source_lines.txt
python tools/ncu_lines.py gpurun_out/r1j_mm1_wlp_10000000.ncu-rep 60 > gpurun_out/round1_mm1_wlp_pipe_source_lines.txt
mkdir -p /tmp/keep && mv gpurun_out/r1j_*.ncu-rep /tmp/keep/ && mv /tmp/keep/r1j_pi_wlp_1000000.ncu-rep gpurun_out/
timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1j_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > gpurun_out/r1j_bench_under_ncu.json 2>&1; echo launches rc=$?
python bench.py > gpurun_out/r1j_bench.json 2> gpurun_out/r1j_bench.err; echo bench rc=$?
