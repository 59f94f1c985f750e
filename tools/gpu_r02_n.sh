export PYTHONPATH=.
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm_tc -s 2 -c 1 \
  -o gpurun_out/r02n_ff1 python tools/bench_linear.py --only bert_b8_ff1 --reps 2 > gpurun_out/r02n.log 2>&1
echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm_tc -s 2 -c 1 \
  -o gpurun_out/r02n_proj python tools/bench_linear.py --only bert_b8_proj_res --reps 2 >> gpurun_out/r02n.log 2>&1
echo rc=$?
timeout 300 python tools/profile_plan.py --model bert-base --instances 8 --batch 1 --out gpurun_out/r02n_timeline_c2.json 2>&1 | head -30
