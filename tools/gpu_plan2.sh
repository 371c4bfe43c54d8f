for r in 0.0 0.7 2.0; do echo "rho=$r"; WLP_MM1_SERIAL_RHO=$r timeout 300 python tools/time_cfg.py mm1:wlp:50000:1000:lambda_=0.9 mm1:wlp:3000:10000:lambda_=0.9 mm1:wlp:3000:10000:lambda_=0.75 mm1:wlp:200000:1000; done
timeout 300 python tools/time_cfg.py mm1:tlp:50000:1000:lambda_=0.9 mm1:tlp:3000:10000:lambda_=0.9
