import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pfac_datagen as gen
import paper_1811_10498_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50 * 1024 + 77
npat = int(sys.argv[2]) if len(sys.argv) > 2 else 300
pats = gen.random_patterns(41, npat, 1, 12)
text = gen.plant(gen.iid_text(41, 0, n), 0, n, pats, 41)
a = P.Automaton(pats)
dev = torch.device("cuda:0")
packed = P.pack_async(torch.from_numpy(text).to(dev))
out = P.match_packed_async(a, packed, n, n); torch.cuda.synchronize()
pos, pid, m = P.compact(out, k=len(pats)); print("separate path ok, matches", m, flush=True)
out2 = torch.empty(n, dtype=torch.int32, device=dev)
pos2 = torch.empty(n + 16, dtype=torch.int64, device=dev); pid2 = torch.empty(n + 16, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
ws = torch.empty(P.compact_workspace_bytes(n), dtype=torch.uint8, device=dev)
P.match_compact_async(a, packed, n, n, out2, pos2, pid2, cnt, ws)
print("launched", flush=True)
torch.cuda.synchronize()
print("fused ok", int(cnt.item()), bool((out2 == out).all()), flush=True)
