import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
from paper_2506_10470_b200 import TDPipe
from workload import SHAPES
shape = SHAPES["llama2_7b"].with_layers(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
t = TDPipe(shape, 1, kv_blocks=int(sys.argv[2]) if len(sys.argv) > 2 else 8000)
t.td_profile("/tmp/p.csv", int(sys.argv[3]) if len(sys.argv) > 3 else 256, 2048, 293)
print("profile ok")
