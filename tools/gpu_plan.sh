timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_plan_gpu.py -q -x -k "mm1 or plan" 2>&1 | tail -2
for r in 0.0 0.5 0.6 0.7 0.8 0.9 2.0; do echo -n "rho=$r "; WLP_MM1_SERIAL_RHO=$r timeout 120 python tools/time_plan.py wlp; done
