# Round 2, call E: new-feature GPU tests, GEMM pipeline traces at C5/C4
# shapes, linear microbench, serving strategies (C2 shape).
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_serving.py tests/test_plan_artifact.py -m gpu -q -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1
tail -3 gpurun_out/r02e_pytest.log
for s in "32 1024 768 2304 none 0" "32 1024 768 768 none 1" "32 1024 768 3072 gelu 0" "32 1024 3072 768 none 1" "32 512 768 3072 gelu 0"; do
  set -- $s
  if [ "$6" = 1 ]; then R=1; else R=; fi
  NF_TRACE_ACT=$5 NF_TRACE_RES=$R timeout 60 tools/bin_gemm_trace $1 $2 $3 $4 2>&1 | head -14
done > gpurun_out/r02e_trace.txt
cat gpurun_out/r02e_trace.txt
timeout 300 python tools/bench_linear.py --only bert_b8_qkv,bert_b8_proj_res,bert_b8_ff1_gelu,bert_b8_ff2_res,bert_b8_ff1,bert_b8_ff2,xlnet_b4_ff1_gelu > gpurun_out/r02e_linear.jsonl 2>&1
cat gpurun_out/r02e_linear.jsonl
timeout 1200 python -m paper_2009_13062_b200.serving --model bert-base --num-models 8 --batch 1 \
  --strategies sequential,concurrent,hybrid:2,hybrid:4,merged --rounds 30 > gpurun_out/r02e_serving_c2.jsonl 2>&1
cat gpurun_out/r02e_serving_c2.jsonl | cut -c1-400
