"""Read the NVML NVLink data counters (TX/RX, all links) of every visible GPU
around a copy between two GPUs: checks that the counters exist and their unit."""
import time

import pynvml as n
import torch

n.nvmlInit()
cnt = n.nvmlDeviceGetCount()
hs = [n.nvmlDeviceGetHandleByIndex(i) for i in range(cnt)]
F = [n.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, n.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]


def read():
    """[gpu] -> [(ret, type, TX sum over links), (ret, type, RX sum)]"""
    out = []
    for h in hs:
        tx = rx = 0
        ret = []
        for link in range(18):
            vals = n.nvmlDeviceGetFieldValues(h, [(f, link) for f in F])
            ret.append(vals[0].nvmlReturn)
            if vals[0].nvmlReturn == 0:
                tx += vals[0].value.ullVal
            if vals[1].nvmlReturn == 0:
                rx += vals[1].value.ullVal
        out.append([(ret[0], 0, tx), (ret[0], 0, rx)])
    return out


print("gpus", cnt, read())
if torch.cuda.device_count() >= 2:
    a = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0")   # 1 GiB
    b = torch.empty(1 << 28, dtype=torch.float32, device="cuda:1")
    r0 = read()
    for _ in range(4):
        b.copy_(a)
    torch.cuda.synchronize("cuda:1")
    torch.cuda.synchronize("cuda:0")
    time.sleep(0.5)
    r1 = read()
    for i in range(cnt):
        print(i, "TX delta", r1[i][0][2] - r0[i][0][2], "RX delta", r1[i][1][2] - r0[i][1][2],
              "(4 GiB copied 0 -> 1)")
