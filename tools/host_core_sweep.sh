# bench --quick with the serving loop pinned to different cores (GMX_HOST_CORE; -1 = unpinned)
for c in ${@:-8 3 15 -1 8}; do
  v=$(GMX_HOST_CORE=$c timeout 300 python bench.py --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_us'])")
  echo "core $c: $v"
done
