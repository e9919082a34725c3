# A/B/C over library builds for cfg4, cfg2, cfg3: bash tools/run_ab3.sh tag lib1 lib2 ...
tag=$1; shift
bash tools/run_ab.sh cfg4 ${tag}4 "$@"
bash tools/run_ab.sh cfg2 ${tag}2 "$@"
bash tools/run_ab.sh cfg3 ${tag}3 "$@"
