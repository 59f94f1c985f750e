# Round evidence: full GPU tests + smoke, bench lines for every BASELINE
# config that fits one GPU, ncu launch list + --set full captures of the
# headline forward (BERT-base N=8 B=1).
export PYTHONPATH=.
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/final_pytest.log 2>&1
tail -3 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench_default.log 2>&1
tail -1 gpurun_out/final_bench_default.log > gpurun_out/final_bench_default.json
for cfg in "xlnet-base 32 4" "resnext50_32x4d 32 1" "resnet50 2 1" "bert-base 32 8" "bert-base 32 1"; do
  set -- $cfg
  timeout 900 python bench.py --steps 30 --warmup 5 --model $1 --instances $2 --batch $3 --no-cpu \
    > gpurun_out/final_bench_$1_N$2_B$3.log 2>&1
  tail -1 gpurun_out/final_bench_$1_N$2_B$3.log > gpurun_out/final_bench_$1_N$2_B$3.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-unmerged \
  > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grouped_gemm_tc|k_qkv_attention" \
  -s 40 -c 6 -o gpurun_out/final_ncu_bert8 python tools/profile_plan.py --model bert-base \
  --instances 8 --batch 1 > /dev/null 2>&1
ls gpurun_out | grep final
