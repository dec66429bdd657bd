# frames/s vs streams / groups with the default (8) and 32 hardware work queues
# (CUDA_DEVICE_MAX_CONNECTIONS; each group uses 3 CUDA streams + the torch stream)
mkdir -p gpurun_out/sweep_conn
for conn in 8 32; do
for cfg in "16 4" "16 8" "24 6" "32 8" "48 12"; do
  set -- $cfg
  CUDA_DEVICE_MAX_CONNECTIONS=$conn timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 --no-quality \
      --streams $1 --groups $2 --steps 12 --warmup 3 \
      > gpurun_out/sweep_conn/c${conn}_s$1_g$2.json 2> gpurun_out/sweep_conn/c${conn}_s$1_g$2.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_conn/c${conn}_s$1_g$2.json')); print('conn $conn streams/groups $cfg', round(d['value']), 'e2e', round(d['e2e']['value']), 'host', d['host_ms_per_step'], 'gen_s', d['input_generation_s'])" || tail -3 gpurun_out/sweep_conn/c${conn}_s$1_g$2.err
done
done
