cd "$GRAFT_REPO_ROOT"
for s in "15000 64 64" "1024 64 47" "129000 100 64"; do for mode in tc3 simt v2; do
  echo "== $s $mode"
  if [ $mode = tc3 ]; then E=""; else E="FGL_DENSE=$mode"; fi
  env $E timeout 60 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 10 python tools/dense_bench.py $s 2>&1 | grep -E "^  [a-z_]|duration" | paste - - | awk '{print $1, $(NF)}' | sort | uniq
done; done
