python tools/phase_probe.py 3 128
for s in "48,4,384,2" "48,4,512,2" "56,4,384,2" "64,4,512,1" "64,8,384,1"; do RD_K2_SHAPE=$s PROBE_ENTRY_CAP=1536 PROBE_HOT_CAP=192 python tools/phase_probe.py 3 128 2>&1; done
