# Round 2, call C: full GPU suite + smoke + default bench + C2 line.
export PYTHONPATH=.
nproc > gpurun_out/r02c_nproc.txt
NF_PARITY_LOG=gpurun_out/r02c_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
  > gpurun_out/r02c_pytest.log 2>&1
tail -15 gpurun_out/r02c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; tail -2 gpurun_out/r02c_smoke.log
timeout 900 python bench.py > gpurun_out/r02c_bench_default.log 2>&1; tail -1 gpurun_out/r02c_bench_default.log | cut -c1-1500
timeout 600 python bench.py --model bert-base --instances 8 --batch 1 --steps 30 --warmup 5 --no-cpu \
  > gpurun_out/r02c_bench_c2.log 2>&1; tail -1 gpurun_out/r02c_bench_c2.log | cut -c1-1500
