# 1-GPU box: bench lines (config C causal / non-causal, config B1), the reference arm, the ncu launch list and
# ncu --set full captures of the attention kernels and the [Q|K|V] GEMM (each after its command ran without ncu)
set -x
timeout 300 python bench.py > gpurun_out/${TAG:-r2f}_bench.json 2> gpurun_out/${TAG:-r2f}_bench.err
timeout 300 python bench.py --seq 8192 > gpurun_out/${TAG:-r2f}_bench_8192.json 2>> gpurun_out/${TAG:-r2f}_bench.err
timeout 300 python bench.py --noncausal > gpurun_out/${TAG:-r2f}_bench_nc.json 2>> gpurun_out/${TAG:-r2f}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG:-r2f}_ref.json 2>> gpurun_out/${TAG:-r2f}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG:-r2f}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG:-r2f}_ncu1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_tc|attn_bwd_tc" -c 2 -o gpurun_out/${TAG:-r2f}_attn python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG:-r2f}_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm_bf16 -c 1 -o gpurun_out/${TAG:-r2f}_gemm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG:-r2f}_ncu3.log 2>&1
