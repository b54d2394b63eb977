import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from kbench import run
for (E, B) in [(3, 8), (0, 128), (0, 32), (12, 24), (12, 96), (8, 16), (4, 8)]:
    run(4096, 14336, E, B, 30)
    if E:
        run(4096, 14336, E, B, 30, base=False)
