"""One rank's share of config 5 row bands, measured on one GPU: the band
filter (with its bounded halo rows already local) for world sizes 2/4/8,
against the whole image / world (the exchange is not included)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads, sharding
H = W = 32768
w = workloads.config5(H, W, device="cuda", param_dtype=torch.float32, image_device="cuda")
f, p = w["f"], [w["size"], w["elong"], w["orient"]]
lut = rb.default_lut()
def timed(fn, reps=2):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
whole = timed(lambda: rb.filter_space_variant_params(f, *p))
print(f"whole image: {whole:.1f} ms")
for world in (2, 4, 8):
    worst = 0.0
    for rank in (0, world // 2):
        band = sharding.band_bounds(H, world)[rank]
        pb = [v[band[0]:band[1]] for v in p]
        t0 = time.perf_counter()
        m = sharding.halo_bound_params(pb[0], lut)
        torch.cuda.synchronize()
        tb = (time.perf_counter() - t0) * 1e3
        n0, n1 = sharding.needed_rows(band, m, H)
        fr = f[n0:n1].contiguous()
        t = timed(lambda: sharding.filter_rows_params(fr, n0, H, *pb, band[0], band[0], band[1] - band[0]))
        worst = max(worst, t + tb)
        print(f"world {world} rank {rank}: halo {n1 - n0 - (band[1] - band[0])} rows, bound {tb:.2f} ms, band {t:.1f} ms")
    print(f"world {world}: whole/world {whole / world:.1f} ms, slowest band {worst:.1f} ms, efficiency {whole / world / worst:.2f}")
