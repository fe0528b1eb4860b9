import os, sys
sys.path.insert(0, ".")
os.environ["NMX_PARTS_MIN"] = str(1 << 20)
import numpy as np
from oracle import netmeter_oracle as orc
from paper_2510_14050_b200 import _lib
s, d = orc.gen_uniform(31, 0, 5 << 20, 1 << 32)
cuts = [0, 3, 1 << 20, 3 << 20, len(s)]
wins = [(s[a:b], d[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
print(_lib.stream_stats9(wins, 1 << 32), orc.stats9_packed(s, d))
