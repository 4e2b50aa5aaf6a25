import json,sys
name=None
for line in open(sys.argv[1]):
    if line.startswith("=="): name=line.strip(); continue
    try: d=json.loads(line)
    except Exception: continue
    r=[k for k in d if k.startswith('adj_c3x')][0].split('x')[1].split('_')[0]
    print(name, "adj %.4f chol %.4f | adj64 %.4f chol64 %.4f" % (d[f"adj_c3x{r}_ms"], d[f"chol_c3x{r}_ms"], d[f"adj_fp64_c3x{r}_ms"], d[f"chol_fp64_c3x{r}_ms"]))
