import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, bench
import paper_1711_05683_b200 as hk
print(json.dumps(bench.splot_pass(hk, torch)))
