set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_bert8.log 2>&1; tail -2 gpurun_out/bench_bert8.log
timeout 600 python bench.py --steps 20 --warmup 5 --model xlnet-base --instances 32 --batch 4 --no-cpu > gpurun_out/bench_xlnet.log 2>&1; tail -2 gpurun_out/bench_xlnet.log
timeout 600 python bench.py --steps 20 --warmup 5 --model resnext50_32x4d --instances 32 --no-cpu > gpurun_out/bench_resnext.log 2>&1; tail -2 gpurun_out/bench_resnext.log
timeout 600 python bench.py --steps 20 --warmup 5 --model resnet50 --instances 2 --no-cpu > gpurun_out/bench_resnet.log 2>&1; tail -2 gpurun_out/bench_resnet.log
