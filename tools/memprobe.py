import sys, torch
sys.path.insert(0, '.')
import paper_1811_03559_b200 as spk
L = spk.lib()
n, k, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device('cuda', 0)
s = torch.cuda.current_stream().cuda_stream
band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
F = torch.empty((r, n), dtype=torch.float64, device=dev); X = torch.empty_like(F)
spk.generate_band_device(1, n, k, k, 1.2, band.data_ptr(), s)
spk.generate_rhs_device(2, n, r, F.data_ptr(), n, s)
def info(tag):
    fr, tot = torch.cuda.mem_get_info()
    print(f"{tag}: free {fr/1e9:.1f} GB, torch reserved {torch.cuda.memory_reserved()/1e9:.1f}, arena cached {L.spk_arena_cached()/1e9:.1f}", flush=True)
info("inputs")
plan = spk.gpu_plan(n, k, k, r)
try:
    f = spk.factorize_device(band.data_ptr(), n, k, k, plan, spk.FactorOptions(), s)
    torch.cuda.synchronize(); info("factored")
    spk.solve_device(f, F.data_ptr(), n, r, X.data_ptr(), n, False, s)
    torch.cuda.synchronize(); info("solved")
except Exception as e:
    print("ERR", e); info("at error")
