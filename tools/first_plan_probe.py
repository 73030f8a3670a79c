"""Where the first tt_plan of a process spends its time (GPU box): context
creation, library load, device query, first occupancy query / module load.
Run twice: default (lazy module loading) and CUDA_MODULE_LOADING=EAGER."""
import ctypes, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
t = {}
t0 = time.perf_counter()
import torch
torch.cuda.init(); torch.empty(1, device="cuda"); torch.cuda.synchronize()
t["torch_ctx_ms"] = (time.perf_counter() - t0) * 1e3
t0 = time.perf_counter()
import paper_1705_01598_b200 as tt
t["import_tt_ms"] = (time.perf_counter() - t0) * 1e3
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
def plan(dims, perm, e, tag):
    t0 = time.perf_counter(); p = tt.Plan(dims, perm, e); dt = (time.perf_counter() - t0) * 1e3
    t[tag] = round(dt, 3); k = p.describe()["kernel"]; p.destroy(); return k
plan((16384, 16384), (1, 0), 4, "plan1_s1_ms")
plan((16384, 16384), (1, 0), 4, "plan2_s1_cached_ms")
plan((300, 200, 77), (1, 0, 2), 4, "plan3_tiled2d_batch_ms")
plan((5,) * 12, (0, 8, 4, 10, 1, 3, 9, 5, 7, 2, 6, 11), 4, "plan4_vg_ms")
plan((7, 13, 12, 11, 5, 5, 3, 3, 7, 3, 4), (2, 3, 6, 5, 8, 0, 10, 9, 7, 4, 1), 8, "plan5_sd8_ms")
plan((2584, 172, 548), (1, 0, 2), 4, "plan6_sd4_ms")
plan((1233, 427, 247), (0, 2, 1), 4, "plan7_rowcopy_ms")
x = torch.empty(1 << 20, dtype=torch.int32, device="cuda"); y = torch.empty_like(x)
p = tt.Plan((1024, 1024), (1, 0), 4)
torch.cuda.synchronize(); t0 = time.perf_counter(); p.execute(x, y); torch.cuda.synchronize()
t["first_execute_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
t0 = time.perf_counter(); p.execute(x, y); torch.cuda.synchronize()
t["second_execute_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
t["CUDA_MODULE_LOADING"] = os.environ.get("CUDA_MODULE_LOADING", "(default)")
print(json.dumps(t))
