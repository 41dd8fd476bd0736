"""PCIe H2D ceiling: pinned 1 GiB on one stream vs split over 2 / 4 streams."""
import torch

torch.cuda.set_device(0)
nb = 1 << 30
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    best = 0
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        part = nb // ns
        for i in range(ns):
            streams[i].wait_event(e0)
            with torch.cuda.stream(streams[i]):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for i in range(ns):
            torch.cuda.current_stream().wait_stream(streams[i])
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nb / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print(f"H2D pinned 1 GiB over {ns} stream(s): {best:.1f} GB/s")
# chunked on one stream (16 MiB pieces)
for piece in (4 << 20, 16 << 20, 64 << 20):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for o in range(0, nb, piece):
        d[o:o + piece].copy_(h[o:o + piece], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"H2D pinned 1 GiB in {piece >> 20} MiB pieces: {nb / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
