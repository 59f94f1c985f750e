# ncu --set full captures of one launch of each top kernel in a merged plan.
# usage: tools/gpu_ncu_bert8.sh <model> <instances> <batch> <tag>
set -x
M=$1; N=$2; B=$3; TAG=$4
export PYTHONPATH=.
for pat in "k_grouped_gemm_tc" "k_group_norm" "attention"; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$pat -s 30 -c 1 \
    -o gpurun_out/ncu_${TAG}_${pat} python tools/profile_plan.py --model $M --instances $N --batch $B > /dev/null 2>&1
done
ls -la gpurun_out/
