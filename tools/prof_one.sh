# ncu of one kernel (CSV on the box): bash tools/prof_one.sh NAME REGEX profile_driver-args...
n=$1; k=$2; shift 2
ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:$k -o /tmp/$n python tools/profile_driver.py "$@" > /dev/null 2>&1
ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/$n.raw.csv 2>&1
ncu -i /tmp/$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$n.src.csv 2>&1
gzip -f gpurun_out/$n.src.csv
