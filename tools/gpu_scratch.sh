export PYTHONPATH=.
NF_GEMM_KPT=3 timeout 600 python -m pytest tests/test_gpu_fold.py tests/test_gpu_linear_smoke.py tests/test_gpu_execute.py -q --timeout 300 -x 2>&1 | tail -2
for shape in "8 128 768 768" "8 128 3072 768" "8 128 768 3072"; do
for k in 2 3; do echo "## kpt=$k $shape warm"; NF_GEMM_KPT=$k NF_TRACE_WARM=1 NF_PDL=0 timeout 60 ./tools/bin/gemm_trace $shape | grep -E "first_stage|last_mma"; done
done
for i in 1 2; do for k in 2 3; do
echo "kpt=$k $(NF_GEMM_KPT=$k timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
done; done
