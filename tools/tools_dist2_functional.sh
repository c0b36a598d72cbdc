# bench.py's N > 1 path on a one-GPU box: 2 ranks sharing GPU 0 over gloo
# (functional check of torchrun launch, barriers, max-over-ranks, gather and
# the reference arm on rank 0; not a measurement).  Also the halo split.
mkdir -p gpurun_out
export CS_BENCH_DIST_BACKEND=gloo CS_BENCH_FORCE_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 4 --warmup 3 --no-parity > gpurun_out/r2_dist2.log 2>&1; echo dist2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 2 --warmup 3 --impl reference > gpurun_out/r2_dist2_ref.log 2>&1; echo dist2ref=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 3 --warmup 3 --c2-split halo > gpurun_out/r2_dist2_halo.log 2>&1; echo dist2halo=$?
for f in r2_dist2 r2_dist2_ref r2_dist2_halo; do tail -1 gpurun_out/$f.log | cut -c1-400; done
