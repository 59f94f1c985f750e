export PYTHONPATH=.
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm_tc -s 2 -c 1 \
  -o gpurun_out/r02l_ff1 python tools/bench_linear.py --only bert_b8_ff1 --reps 2 > gpurun_out/r02l.log 2>&1
echo rc=$?; tail -2 gpurun_out/r02l.log
