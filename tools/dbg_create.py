"""Create a detector for the dense cfg4 capacities and print rd_create's error, if any (RD_K2_VERBOSE=1 shows the K2 shape)."""
import os, sys
sys.path.insert(0, os.getcwd())
import synth, paper_1310_1371_b200 as rd
from paper_1310_1371_b200 import _rd
params = dict(synth.preset(4), max_entries_per_tile=6144, max_hotspots_per_level=512)
try:
    det = rd.Detector(params, max_batch=512)
    print("ok")
except Exception as e:
    print("ERR", e, _rd.lib().rd_last_error())
