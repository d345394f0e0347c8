# 4-GPU box: NCCL dist tests, then N=1/2/4 bench lines (one rank per GPU, no oversubscription)
set -x
T=${TAG:-r2m}
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/${T}_dist.log 2>&1; echo exit=$? >> gpurun_out/${T}_dist.log
timeout 300 python bench.py > gpurun_out/${T}_n1.json 2> gpurun_out/${T}_n1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/${T}_n2.json 2> gpurun_out/${T}_n2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/${T}_n4.json 2> gpurun_out/${T}_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 4 > gpurun_out/${T}_ref_n4.json 2> gpurun_out/${T}_ref_n4.err
