# round-2 capture: microbench + ncu full of the config-4 kernels; reports are reduced to
# CSV (raw metrics + source page) on the box to stay under gpurun's copy-back limit
./tools/microbench > gpurun_out/microbench.txt 2>&1
P="ncu --set full --clock-control none --import-source on -s 1 -c 1"
run() {  # name regex args...
  n=$1; k=$2; shift 2
  $P -k regex:$k -o /tmp/$n python tools/profile_driver.py "$@" > /dev/null 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/$n.raw.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$n.src.csv 2>&1
  gzip -f gpurun_out/$n.src.csv
}
run r2_pi_wlp k_wlp_pipe pi wlp 10000000 1000
run r2_pi_tlp k_tlp pi tlp 10000000 1000
run r2_walk_wlp k_wlp_walk_bs_pipe walk wlp 10000000 1000
run r2_walk_tlp k_tlp_walk_bs walk tlp 10000000 1000 --tlp-variant 2
run r2_mm1_wlp k_wlp_mm1_pipe mm1 wlp 10000000 1000
ls -la gpurun_out
