cp paper_2310_10211_b200/libgevo.so /tmp/libgevo_main.so
cp tests/tools/_build/libgevo_timing.so paper_2310_10211_b200/libgevo.so
cd tests/tools
for a in "bigsgd 32" "bigsgd 296" "small 32" "small 296"; do echo "== $a"; python dot_phase.py $a; done
cd ../..; cp /tmp/libgevo_main.so paper_2310_10211_b200/libgevo.so
