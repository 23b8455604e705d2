# A/B on one box: libs under _ab/ (lib<X>.so) vs the in-tree build (B)
LIBS=${LIBS:-A}
for r in 1 2; do
for X in $LIBS; do echo "$X"; LINKSDF_B200_LIB=_ab/lib$X.so python tools/stage_times.py --workload config4 --n 30 | grep graph; done
echo "B"; python tools/stage_times.py --workload config4 --n 30 | grep graph
done
for X in $LIBS; do echo "$X c2"; LINKSDF_B200_LIB=_ab/lib$X.so python tools/latency_parts.py 2>/dev/null | tail -1; done
echo "B c2"; python tools/latency_parts.py 2>/dev/null | tail -1
