cd "$GRAFT_REPO_ROOT"; O=gpurun_out/$1; mkdir -p $O
for d in 8 9 10 12 13 15; do
 echo "dbg=$d" >> $O/exp.log
 FGL_G3DBG=$d timeout 60 python tools/g3_trace.py 2>&1 | sed -n '2,9p;$p' >> $O/exp.log
done
cat $O/exp.log
