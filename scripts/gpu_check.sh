set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python -c "import torch;print(torch.cuda.get_device_properties(0))"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not config2_full and not config5_full" 2>&1 | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -5
