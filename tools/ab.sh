# usage: ab.sh tag lib1 lib2 ... ; runs bench twice per lib interleaved
tag=$1; shift
for k in 1 2; do for L in "$@"; do n=$(basename $L .so); MPSKQ_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/ab_${tag}_${n}_$k.json 2>/dev/null; done; done
for f in gpurun_out/ab_${tag}_*.json; do python -c "import json,sys; d=json.load(open(\"$f\")); print(\"$f\", round(d[\"phases_ms\"][\"overlap\"],2), round(d[\"roofline\"][\"frac\"],4), round(d[\"e2e\"][\"ms_per_step\"],2))"; done
