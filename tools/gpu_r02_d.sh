# Round 2, call D: per-config ncu launch lists (+DRAM bytes), --set full
# captures of each config's top kernel, bench lines C1-C4, sanitizer.
export PYTHONPATH=.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for C in C1 C2 C3 C4 C5; do
  timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file gpurun_out/r02_ncu_$C.csv python tools/ncu_forward.py --config $C \
    --meta gpurun_out/r02_ncu_${C}_meta.json > gpurun_out/r02_ncu_$C.log 2>&1
  echo "ncu $C rc=$? $(grep -c k_ gpurun_out/r02_ncu_$C.csv)"
done
full() {  # config regex count out
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"$2" -c $3 -o gpurun_out/r02_full_$4 python tools/ncu_forward.py --config $1 \
    > gpurun_out/r02_full_$4.log 2>&1; echo "full $4 rc=$?"
}
full C5 k_grouped_gemm_tc 4 c5_gemm
full C5 "k_attention_tc|k_group_norm" 2 c5_attn_norm
full C3 k_grouped_gemm_tc 6 c3_conv
full C4 "k_rel_attention|k_grouped_gemm_tc" 5 c4
full C1 k_conv_tf32 4 c1_conv
full C2 "k_grouped_gemm_tc|k_qkv" 4 c2
for C in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $C > gpurun_out/r02d_bench_$C.log 2>&1
  echo "bench $C rc=$?"; tail -1 gpurun_out/r02d_bench_$C.log | cut -c1-300
done
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_linear_smoke.py tests/test_gpu_conv_igemm.py tests/test_gpu_fold.py tests/test_gpu_conv_tf32.py -q -p no:cacheprovider \
    > gpurun_out/r02d_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r02d_sanitizer_$tool.log
done
