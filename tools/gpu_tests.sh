timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_gpu.log
