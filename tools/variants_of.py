"""Print the global indices of the compiled variants of (kind, tb): python tools/variants_of.py K TB"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g
k, tb = int(sys.argv[1]), int(sys.argv[2])
print(" ".join(str(v["index"]) for v in g.variants() if v["kind"] == k and v["tb"] == tb))
