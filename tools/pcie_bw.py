"""Experiment: H2D bandwidth from pinned memory for the end-to-end step's
copy pattern (4 x 8 MB parameter arrays + 8 x (2.4 + 1.6 MB) frames) vs one
coalesced 65 MB copy, alone and under a concurrent compute kernel load."""
import torch


def bw(copies, reps=10, stream=None):
    s = stream or torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for d, h in copies:
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(reps):
            for d, h in copies:
                d.copy_(h, non_blocking=True)
        b.record(s)
    torch.cuda.synchronize()
    nbytes = sum(h.numel() * h.element_size() for _, h in copies) * reps
    return nbytes / (a.elapsed_time(b) * 1e-3) / 1e9


def pair(nbytes):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    return torch.empty(nbytes, dtype=torch.uint8, device="cuda"), h


pattern = [pair(8_000_000) for _ in range(4)] + [pair(48 * 8)]
for _ in range(8):
    pattern += [pair(1200 * 680 * 3), pair(1200 * 680 * 2)]
big = [pair(sum(h.numel() for _, h in pattern))]
print("pattern (%d copies): %.1f GB/s" % (len(pattern), bw(pattern)))
print("one coalesced copy:  %.1f GB/s" % bw(big))
