import json, os, sys
sys.path.insert(0, os.getcwd())
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
qs = [Query.from_json(d["query"]) for d in json.load(open("synth/data/cfg2_queries.json"))["queries"]]
ctx = gpsense.Context(0, workers=1)
ctx.set_slice(100)
G = ctx.load_graph(config_graph(2))
ctx.count_batch(G, qs)
ctx.close()
