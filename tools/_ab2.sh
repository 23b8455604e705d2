# latency A/B: lib A (_ab/libA.so) vs in-tree B, interleaved
for i in 1 2 3; do
  echo A; LINKSDF_B200_LIB=_ab/libA.so python tools/latency_parts.py 2>/dev/null | grep -E "^query|checker"
  echo B; python tools/latency_parts.py 2>/dev/null | grep -E "^query|checker"
done
