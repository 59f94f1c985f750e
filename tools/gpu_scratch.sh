export PYTHONPATH=.
NF_GEMM_KPT=2 timeout 600 python -m pytest tests/test_gpu_fold.py tests/test_gpu_linear_smoke.py tests/test_gpu_execute.py -q --timeout 300 -x 2>&1 | tail -3
for i in 1 2; do
echo "kpt2 fold $(NF_GEMM_KPT=2 timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
echo "kpt1 fold $(timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
echo "kpt2 B32  $(NF_GEMM_KPT=2 timeout 120 python bench.py --no-unmerged --no-cpu --instances 32 2>&1 | tail -1 | cut -c150-210)"
echo "kpt1 B32  $(timeout 120 python bench.py --no-unmerged --no-cpu --instances 32 2>&1 | tail -1 | cut -c150-210)"
done
