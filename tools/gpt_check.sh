# 4-GPU box: whole-decoder steps (BASELINE configs 4/5 shapes at 4 GPUs), then the full GPU suite and smoke()
set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --model gpt --gpus 4 --seq 32768 --batch 4 --steps 3 --warmup 3 > gpurun_out/${TAG:-r2g}_cfg5_replica.json 2> gpurun_out/${TAG:-r2g}_gpt.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --model gpt --gpus 4 --replicas 2 --seq 32768 --batch 4 --steps 3 --warmup 3 > gpurun_out/${TAG:-r2g}_2x2.json 2>> gpurun_out/${TAG:-r2g}_gpt.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG:-r2g}_gpu_pytest.log 2>&1; echo exit=$? >> gpurun_out/${TAG:-r2g}_gpu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG:-r2g}_smoke.log 2>&1
