"""Check whether gen.c1_dense reproduces the reference run's input bytes here
(the C1 goldens were recorded in the build container)."""
import hashlib, json, os, sys
sys.path.insert(0, os.getcwd())
from threadpoolctl import threadpool_info
from paper_2601_22344_b200 import gen
print([(d['internal_api'], d.get('architecture'), d.get('num_threads')) for d in threadpool_info()])
runs = {r["seed"]: r for r in json.load(open("tests/golden/c1_reference.json"))["runs"]}
ok = 0
for s in range(30):
    A = gen.c1_dense(s)
    ok += hashlib.sha256(A.tobytes()).hexdigest() == runs[s]["sha256"]
print("match", ok, "/30")
