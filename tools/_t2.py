import sys, json
sys.path.insert(0, ".")
from tools.time_asm import run
for c in [(2, 5, 256, 2, 0), (2, 5, 256, 2, 8), (2, 6, 256, 2, 0), (2, 4, 256, 2, 8), (3, 2, 64, 3, 0)]:
    print(json.dumps(run(*c, reps=20)))
