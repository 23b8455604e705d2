# A/B on one box: _ab/lib<X>.so for X in $LIBS (default A B), scan + cycle, L2 flushed
for r in 1 2; do
  for X in ${LIBS:-A B}; do echo $X; LINKSDF_B200_LIB=_ab/lib$X.so python tools/_scan_timing.py ${W:-config4 config2} | grep flushed; done
done
