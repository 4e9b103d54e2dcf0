import json, sys
for l in open(sys.argv[1]):
    try:
        g = json.loads(l)
    except Exception:
        continue
    print("div=" + sys.argv[2], g["graph"], round(g["score_ms"], 3), "cluster",
          round(g["score_cluster_ms"] - g["score_ms"], 3), "kept", g["kept"])
