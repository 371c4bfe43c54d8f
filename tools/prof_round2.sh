#!/bin/bash
# Round-2 evidence on the GPU box (writes CSV only, so gpurun can copy it back):
#  * the launch list of a short bench run (per-launch gpu__time_duration, --clock-control none)
#  * ncu --set full of every config's model kernels, reduced to the raw page (CSV) and the
#    source page (CSV, gzip) on the box
#   bash tools/prof_round2.sh OUTDIR [capture names...]   (no names: the launch list and all)
out=${1:-gpurun_out/r2}
shift
only="$*"
mkdir -p $out
if [ -z "$only" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > $out/launches_bench.stdout 2>&1
fi
cap() {  # label kernel-regex profile_driver args...
  n=$1; k=$2; shift 2
  if [ -n "$only" ] && [[ " $only " != *" $n "* ]]; then return; fi
  ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:$k -o /tmp/$n \
      python tools/profile_driver.py "$@" > $out/$n.stdout 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $out/$n.raw.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > $out/$n.src.csv.gz
  rm -f /tmp/$n.ncu-rep
}
cap cfg2_pi_wlp 'k_wlp_pipe' pi wlp 1000000 10000
cap cfg2_pi_tlp '^k_tlp$' pi tlp 1000000 10000
cap cfg3_walk_wlp 'k_wlp_walk_bs_lanes' walk wlp 100000 1000
cap cfg3_walk_tlp '^k_tlp$' walk tlp 100000 1000
cap cfg3_seed 'k_seed' walk wlp 100000 1000
cap cfg4_seed 'k_seed' pi wlp 10000000 1000
cap cfg4_seed_walk_planes 'k_seed' walk wlp 10000000 1000
cap cfg4_pi_wlp 'k_wlp_pipe' pi wlp 10000000 1000
cap cfg4_pi_tlp '^k_tlp$' pi tlp 10000000 1000
cap cfg4_mm1_wlp 'k_wlp_mm1_pipe' mm1 wlp 10000000 1000
cap cfg4_mm1_tlp 'k_tlp_mm1' mm1 tlp 10000000 1000
cap cfg4_walk_wlp 'k_wlp_walk_bs_pipe' walk wlp 10000000 1000
cap cfg4_walk_tlp_bs 'k_tlp_walk_bs' walk tlp 10000000 1000 --tlp-variant 2
cap cfg4_walk_wlp_perrep 'k_wlp_pipe' walk wlp 10000000 1000 --wlp-variant 2
cap cfg4_walk_tlp '^k_tlp$' walk tlp 10000000 1000
# config 5 plans (tools/time_plan_overhead.py runs the mm1 plan, then the walk plan)
capp() {
  n=$1; k=$2
  if [ -n "$only" ] && [[ " $only " != *" $n "* ]]; then return; fi
  ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:$k -o /tmp/$n \
      python tools/time_plan_overhead.py > $out/$n.stdout 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $out/$n.raw.csv 2>&1
  rm -f /tmp/$n.ncu-rep
}
capp cfg5_plan_mm1 'k_plan_mm1'
capp cfg5_plan_walk 'k_plan_lanes'
ls -la $out
