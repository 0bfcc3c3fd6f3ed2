# A/B of whole-library variants: tools/ab/<X>.so swapped in for libnsm.so, config-4 step time (CUDA graph) by chunk_time.py
L=paper_2301_05262_b200/libnsm.so
cp $L /tmp/libnsm.keep
for r in 1 2; do
for X in "$@"; do
  cp tools/ab/$X.so $L
  echo -n "$X: "; timeout 300 python tools/chunk_time.py 2>&1 | tail -1
done
done
cp /tmp/libnsm.keep $L
