# K2 tile-size A/B on cfg3: args "T,G,threads,ctas:hot_cap:entry_cap" ...
export RD_K2_VERBOSE=1
for a in "$@"; do
  IFS=: read s hc ec <<< "$a"
  RD_K2_SHAPE2=$s PROBE_HOT_CAP=$hc PROBE_ENTRY_CAP=$ec python tools/phase_probe.py 3 128 2>&1 | grep -E "us/frame|rd: K2" | sed "s/^/$a /"
done
