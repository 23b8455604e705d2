# A/B on one box: A = _ab/libA.so, B = in-tree build
for r in 1 2; do
echo "A"; LINKSDF_B200_LIB=_ab/libA.so python tools/stage_times.py --workload config4 --n 30 | grep graph
echo "B"; python tools/stage_times.py --workload config4 --n 30 | grep graph
done
echo "A c2"; LINKSDF_B200_LIB=_ab/libA.so python tools/latency_parts.py 2>/dev/null | tail -1
echo "B c2"; python tools/latency_parts.py 2>/dev/null | tail -1
