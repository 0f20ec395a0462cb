mkdir -p gpurun_out/r01n
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-cpu > gpurun_out/r01n/bench_2rank_gloo.json 2> gpurun_out/r01n/bench_2rank_gloo.err
echo "rc=$?" >> gpurun_out/r01n/bench_2rank_gloo.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-dedup > gpurun_out/r01n/bench_1rank_torchrun.json 2> gpurun_out/r01n/bench_1rank_torchrun.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01n/bench_reference.json 2> gpurun_out/r01n/bench_reference.err
cat gpurun_out/r01n/*.json; tail -3 gpurun_out/r01n/bench_2rank_gloo.err
