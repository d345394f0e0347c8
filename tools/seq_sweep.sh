# 1-GPU box: the layer step at several sequence lengths (causal, E=1024, 16 heads), N=1
for L in 8192 16384 32768 50112 65536 131072; do
  timeout 300 python bench.py --seq $L --no-cpu-baseline > gpurun_out/${TAG:-r2s}_seq_$L.json 2>/dev/null
done
