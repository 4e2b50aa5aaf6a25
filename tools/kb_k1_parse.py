import json,sys
name=None
for line in open(sys.argv[1]):
    if line.startswith("=="): name=line.strip(); continue
    try: d=json.loads(line)
    except Exception: print(line[:200]); continue
    print(name, "chol c3 %.3f ms %.0f GB/s | adj %.3f | chol64 %.3f" % (d["chol_c3x5000_ms"], d["chol_c3x5000_GBps"], d["adj_c3x5000_ms"], d["chol_fp64_c3x5000_ms"]))
