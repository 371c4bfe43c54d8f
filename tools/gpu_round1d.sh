timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench_rc=$?; tail -3 gpurun_out/bench4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-extras --no-cpu > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo torchrun_rc=$?; tail -3 gpurun_out/bench_torchrun1.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?; tail -2 gpurun_out/bench_ref.err
