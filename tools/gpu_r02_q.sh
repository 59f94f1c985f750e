export PYTHONPATH=.
for v in base noldsw bfe077d 07138af; do
  if [ $v = base ]; then L=; else L=varlib/lib_$v.so; fi
  echo "== $v $(NF_LIB_PATH=$L timeout 300 python tools/ab_plan.py --config C2 --variants fuse=1 --steps 50 2>&1 | tail -1)"
done
timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_plan_artifact.py -q -p no:cacheprovider > gpurun_out/r02q_pytest.log 2>&1; tail -3 gpurun_out/r02q_pytest.log
NF_PARITY_LOG=gpurun_out/r02q_parity.jsonl timeout 900 python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider -k "C3 or C1" > gpurun_out/r02q_configs.log 2>&1; tail -3 gpurun_out/r02q_configs.log
timeout 300 python tools/ab_plan.py --config C3 --variants fuse=1 2>&1 | tail -1
