# A/B of two libgmx_exec.so builds on C1 (tools/configs.py): old = $1 (default _ab_old/), new = in-tree
OLD=${1:-_ab_old/libgmx_exec.so}
for v in old new old new; do
  LIB=""; [ $v = old ] && LIB="--exec-lib $OLD"
  echo "== $v" >> gpurun_out/c1.log
  python tools/configs.py --configs c1 --rounds 200 $LIB >> gpurun_out/c1.log 2>&1
  python tools/configs.py --configs c1 --rounds 200 --resident $LIB >> gpurun_out/c1.log 2>&1
done
