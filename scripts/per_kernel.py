import json,sys
d=json.loads(sys.stdin.read()); print(sys.argv[1], d["value"], {k:v["gbs"] for k,v in d["per_kernel"].items()})
