import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from _harness import Gpu, inputs
c = inputs("C2", begin=0, end=512)
g = Gpu("C2").run(c)
print("ok", g["o"][:, :3])
