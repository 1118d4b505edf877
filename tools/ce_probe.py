"""What waits behind a large D2H copy running on another stream?  (copy-engine probe)"""
import time, torch
dev = torch.device("cuda", 0)
big = torch.empty(12 * 1024**3, dtype=torch.uint8, device=dev)
hbig = torch.empty(12 * 1024**3, dtype=torch.uint8).pin_memory()
small = torch.ones(8, dtype=torch.float64, device=dev)
hsmall_pinned = torch.empty(8, dtype=torch.float64).pin_memory()
hin = torch.empty(143 * 1024**2, dtype=torch.uint8).pin_memory()
din = torch.empty_like(hin, device=dev)
s = torch.cuda.Stream()
def t(f, name):
    torch.cuda.current_stream().synchronize()
    t0 = time.perf_counter(); f(); torch.cuda.current_stream().synchronize()
    print(f"  {name}: {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
def ops(tag):
    print(tag)
    t(lambda: small.add_(1.0), "kernel")
    t(lambda: small.cpu(), "small D2H pageable")
    t(lambda: hsmall_pinned.copy_(small, non_blocking=True), "small D2H pinned async")
    t(lambda: din.copy_(hin, non_blocking=True), "H2D 143 MB pinned")
    t(lambda: torch.empty(1 << 28, dtype=torch.uint8, device=dev), "alloc 256 MB")
ops("idle")
for mode in ("one copy", "chunks 4 MB all queued", "chunks 4 MB paced depth 2"):
    torch.cuda.synchronize()
    if mode == "one copy":
        with torch.cuda.stream(s):
            hbig.copy_(big, non_blocking=True)
        ops("during " + mode)
    elif mode.endswith("queued"):
        with torch.cuda.stream(s):
            for o in range(0, big.numel(), 4 << 20):
                hbig[o:o + (4 << 20)].copy_(big[o:o + (4 << 20)], non_blocking=True)
        ops("during " + mode)
    else:
        import threading
        def worker():
            evs = [torch.cuda.Event(), torch.cuda.Event()]
            with torch.cuda.stream(s):
                for q, o in enumerate(range(0, big.numel(), 4 << 20)):
                    if q >= 2:
                        evs[q % 2].synchronize()
                    hbig[o:o + (4 << 20)].copy_(big[o:o + (4 << 20)], non_blocking=True)
                    evs[q % 2].record(s)
            s.synchronize()
        th = threading.Thread(target=worker); t0 = time.perf_counter(); th.start()
        time.sleep(0.01)
        ops("during " + mode)
        th.join(); print(f"  copy thread done after {1e3*(time.perf_counter()-t0):.1f} ms")
    t0 = time.perf_counter(); s.synchronize(); print(f"  remaining copy {1e3*(time.perf_counter()-t0):.1f} ms")
