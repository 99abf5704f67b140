import json, sys
d = json.loads(sys.stdin.read())
r = d["roofline"]
print(sys.argv[1], "kernel_ms %.4f frac %.3f" % (r["kernel_ms"], r["frac"]))
