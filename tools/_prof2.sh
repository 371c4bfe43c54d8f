# ncu of the pi / walk warp pipelines at config 4 by lanes per replication (CSV on the box)
P="ncu --set full --clock-control none --import-source on -s 1 -c 1"
run() {  # name regex args...
  n=$1; k=$2; shift 2
  $P -k regex:$k -o /tmp/$n python tools/profile_driver.py "$@" > /dev/null 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/$n.raw.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$n.src.csv 2>&1
  gzip -f gpurun_out/$n.src.csv
}
python tools/time_cfg.py pi:wlp:10000000:1000:wv=2:pl=32 pi:wlp:10000000:1000:wv=2:pl=16 pi:wlp:10000000:1000:wv=2:pl=8 walk:wlp:10000000:1000:wv=2:pl=32 walk:wlp:10000000:1000:wv=2:pl=8 pi:tlp:10000000:1000 pi:wlp:1000000:10000 pi:tlp:1000000:10000
run r2b_pi_s8 k_wlp_pipe pi wlp 10000000 1000 --wlp-variant 2 --pipe-lanes 8
run r2b_pi_s32 k_wlp_pipe pi wlp 10000000 1000 --wlp-variant 2 --pipe-lanes 32
