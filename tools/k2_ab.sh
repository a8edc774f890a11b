# A/B of the Hough kernel shapes on cfg3 via phase_probe (args: shapes "G,threads,ctas" ...)
export RD_K2_VERBOSE=1
for s in "$@"; do RD_K2_SHAPE2=$s python tools/phase_probe.py 3 128 2>&1 | grep -v "CTAs 0" | sed "s/^/v2-$s /"; done
