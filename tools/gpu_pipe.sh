timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "variant or pipeline or full_size or golden" > gpurun_out/pytest_pipe.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_pipe.log
timeout 300 python tools/time_cfg.py pi:wlp:10000000:1000 pi:tlp:10000000:1000 walk:wlp:10000000:1000 walk:tlp:10000000:1000 pi:wlp:1000000:10000 walk:wlp:100000:1000 2>&1 | tee gpurun_out/time_pipe.txt
