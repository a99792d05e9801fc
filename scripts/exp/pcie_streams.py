"""PCIe throughput with 1/2/4 concurrent copy streams per direction (pinned
host memory, 2 GiB per direction): does more than one DMA stream raise the
e2e ceiling?"""
import time

import torch

N = 2 << 30
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 8):
    for mode in ("h2d", "d2h", "duplex"):
        streams = [torch.cuda.Stream() for _ in range(2 * k)]
        chunk = N // k
        best = 0.0
        for rep in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for i in range(k):
                if mode in ("h2d", "duplex"):
                    with torch.cuda.stream(streams[i]):
                        d_in[i * chunk:(i + 1) * chunk].copy_(h_in[i * chunk:(i + 1) * chunk], non_blocking=True)
                if mode in ("d2h", "duplex"):
                    with torch.cuda.stream(streams[k + i]):
                        h_out[i * chunk:(i + 1) * chunk].copy_(d_out[i * chunk:(i + 1) * chunk], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            gb = (2 if mode == "duplex" else 1) * N / dt / 1e9
            best = max(best, gb)
        print(f"streams/dir={k} {mode}: {best:.1f} GB/s", flush=True)
