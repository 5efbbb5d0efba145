# Decomposition checks on one GPU: decomposition tests (local pack / fused /
# fused-concurrent, IPC peer processes) and the N>1 bench path with every
# rank on cuda:0 (FKC_BENCH_ONE_DEVICE=1, timings meaningless).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests/test_decomp.py -m gpu -q -x > gpurun_out/pytest_decomp.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_decomp.txt
FKC_BENCH_ONE_DEVICE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --grid-n 2048 > gpurun_out/bench_onedev2.txt 2>&1; echo "rc=$?" >> gpurun_out/bench_onedev2.txt
FKC_BENCH_ONE_DEVICE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 20 --warmup 3 --grid-n 1024 > gpurun_out/bench_onedev4.txt 2>&1; echo "rc=$?" >> gpurun_out/bench_onedev4.txt
tail -15 gpurun_out/pytest_decomp.txt; tail -3 gpurun_out/bench_onedev2.txt; tail -3 gpurun_out/bench_onedev4.txt
