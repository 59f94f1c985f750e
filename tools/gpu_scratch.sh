# per-launch timeline evidence for the batch-1 headline (profiles/r01_bert8_timeline.txt)
export PYTHONPATH=.
echo "## tools/profile_plan.py --no-pdl (serialised per-kernel durations, one forward)"
timeout 300 python tools/profile_plan.py --no-pdl 2>&1 | grep -v -i warn
echo; echo "## tools/profile_plan.py (PDL, as benchmarked) + tools/timeline_ends.py (critical-path share per kernel)"
timeout 300 python tools/profile_plan.py 2>&1 | grep -v -i warn | head -1
python tools/timeline_ends.py
for shape in "8 128 768 768" "8 128 768 3072" "8 128 3072 768"; do
echo; echo "## tools/gemm_trace.cu $shape (per-CTA phase times, cold HBM, PDL off)"
NF_PDL=0 ./tools/bin/gemm_trace $shape
echo "## same, operands L2-resident (NF_TRACE_WARM=1)"
NF_TRACE_WARM=1 NF_PDL=0 ./tools/bin/gemm_trace $shape | tail -8
done
