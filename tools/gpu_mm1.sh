timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "mm1 or golden or medium or pins or shards" > gpurun_out/pytest_mm1.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_mm1.log
timeout 300 python tools/time_cfg.py mm1:wlp:10000000:1000 mm1:tlp:10000000:1000 mm1:wlp:1000000:1000 mm1:wlp:1000000:1000:lambda_=0.95 mm1:tlp:1000000:1000:lambda_=0.95 2>&1 | tee gpurun_out/time_mm1.txt
