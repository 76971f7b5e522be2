# A/B two library builds on the bench and dot micro-bench (tool)
# usage: bash tests/tools/ab_lib.sh <alt.so>
ALT=$1
python tests/tools/dot_bench.py small; python tests/tools/dot_bench.py big
python bench.py --steps 3 --warmup 2 --no-cpu-baseline | grep -o '"value": [0-9.]*' | head -2
cp paper_2310_10211_b200/libgevo.so /tmp/libgevo_main.so; cp $ALT paper_2310_10211_b200/libgevo.so
echo "== $ALT"
python tests/tools/dot_bench.py small; python tests/tools/dot_bench.py big
python bench.py --steps 3 --warmup 2 --no-cpu-baseline | grep -o '"value": [0-9.]*' | head -2
cp /tmp/libgevo_main.so paper_2310_10211_b200/libgevo.so
