# Small-Q chain diagnostics: per-kernel timeline (VRS_LIB=tl: an -DVRS_TC_TIMING build) of
# the cells named on the command line ("workload sel q" triples).
# usage: bash tools/diag_small_q.sh "c3 0.1 1" "c4 0.05 1" ...
for cell in "$@"; do
  set -- $cell
  n=""; [ "$1" = c4 ] && n="--n 6250000"; [ "$1" = c5 ] && n="--n 2500000"
  VRS_LIB=tl timeout 300 python tools/tc_timeline.py --workload $1 --sel $2 --q $3 $n 2>&1 | grep -v '^ *wave\|pdl wait\|drain'
done
