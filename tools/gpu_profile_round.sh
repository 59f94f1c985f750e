# Round evidence for the headline workload (BERT-base merged N=8, B=1):
#  1. bench.py default line            -> gpurun_out/bench_default.json
#  2. ncu launch list of bench.py      -> gpurun_out/launches.csv
#  3. ncu --set full on one forward's merged-Linear launches (4 = qkv, proj, ff1, ff2)
#  4. ncu --set full on attention / norm of the same forward
export PYTHONPATH=.
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
tail -1 gpurun_out/bench_default.log > gpurun_out/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-unmerged \
  > /dev/null 2>&1
# profile_plan: 5 warm replays then 3 profiled; skip the first forward's launches
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm_tc \
  -s 49 -c 4 -o gpurun_out/ncu_bert8_gemm python tools/profile_plan.py --model bert-base \
  --instances 8 --batch 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attention|group_norm" \
  -s 36 -c 3 -o gpurun_out/ncu_bert8_attn_norm python tools/profile_plan.py --model bert-base \
  --instances 8 --batch 1 > /dev/null 2>&1
ls -la gpurun_out
