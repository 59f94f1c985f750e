export PYTHONPATH=.
for i in 1 2 3; do
echo "cur  $(timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
echo "prev $(cd tools/bin/prevtree && PYTHONPATH=. timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
done
