set -x
free -g; nproc; cat /proc/cpuinfo | grep "model name" | head -1; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/p1_cfg5.json 2>gpurun_out/p1_cfg5.err
cat gpurun_out/p1_cfg5.json
