"""Where the e2e time of a host-I/O decode step goes (cfg3): graph replay + sync with and
without the host copies, an empty graph, and host-side overhead. Diagnostic only."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    from paper_2502_06766_b200.decoder import TopkDecoder

    cfg = bench.CONFIGS["cfg3"]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 64, 0, dev)
    dec = TopkDecoder(K, V, n, cfg["k"], max_ctx=n)
    qh = q.cpu()
    kh = torch.randn(1, 8, 128).bfloat16()
    vh = torch.randn(1, 8, 128).bfloat16()

    def timeit(fn, steps=100):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / steps * 1e6

    print(f"e2e step (q, k, v host -> out host): {timeit(lambda: dec.step(qh, kh, vh, return_idx=False)):.1f} us")
    print(f"e2e step (q host only):              {timeit(lambda: dec.step(qh, return_idx=False)):.1f} us")
    qp, kp, vp = qh.pin_memory(), kh.pin_memory(), vh.pin_memory()
    print(f"e2e step, pinned q/k/v read in place: {timeit(lambda: dec.step(qp, kp, vp, return_idx=False)):.1f} us")
    print(f"e2e step (q, k, v host, again):      {timeit(lambda: dec.step(qh, kh, vh, return_idx=False)):.1f} us")
    print(f"e2e step, pinned again:              {timeit(lambda: dec.step(qp, kp, vp, return_idx=False)):.1f} us")
    g = dec._graphs[(True, False)]
    print(f"graph replay + sync only:            {timeit(lambda: (g.replay(), torch.cuda.current_stream().synchronize())):.1f} us")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        g.replay()
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph replay back-to-back (device):  {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
    eg = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    x = torch.zeros(1, device=dev)
    with torch.cuda.stream(s):
        with torch.cuda.graph(eg, stream=s):
            x.add_(1)
    print(f"tiny graph replay + sync:            {timeit(lambda: (eg.replay(), torch.cuda.current_stream().synchronize())):.1f} us")
    qd, kd, vd = q, kh.to(dev), vh.to(dev)
    print(f"device-resident step (no copies):    {timeit(lambda: dec.attend(qd)):.1f} us (wall, async)")


if __name__ == "__main__":
    main()
