timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?; tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
