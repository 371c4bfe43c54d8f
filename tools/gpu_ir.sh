timeout 600 python -m pytest tests/test_ir_gpu.py -q -x --timeout 300 > gpurun_out/pytest_ir.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/pytest_ir.log
