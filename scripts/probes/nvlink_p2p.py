"""NVLink peer-to-peer copy bandwidth between the visible GPUs (needs >= 2).

    python scripts/probes/nvlink_p2p.py [--mib 1024] [--json OUT]

For every ordered pair (i, j) with peer access: a device-to-device copy of
--mib MiB from cuda:i to cuda:j, best of 5, timed with CUDA events on the
source device's stream (unidirectional GB/s); then i <-> j both ways at once.
bench.py's multi-GPU line reads the same measurement (p2p_gbs) as the
denominator of its NVLink fraction when it runs on several GPUs.
"""
import argparse
import json
import sys

import torch


def p2p_gbs(src, dst, mib=1024, reps=5):
    """Unidirectional copy bandwidth cuda:src -> cuda:dst in GB/s (None without peer access)."""
    if src == dst or not torch.cuda.can_device_access_peer(src, dst):
        return None
    n = mib * (1 << 20) // 4
    a = torch.empty(n, dtype=torch.float32, device=f"cuda:{src}")
    b = torch.empty(n, dtype=torch.float32, device=f"cuda:{dst}")
    b.copy_(a)  # warm-up: establishes the peer mapping
    torch.cuda.synchronize(src)
    torch.cuda.synchronize(dst)
    best = float("inf")
    with torch.cuda.device(src):
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a, non_blocking=True)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
    return a.numel() * 4 / (best / 1e3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--json")
    args = ap.parse_args()
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"p2p": None, "why": f"{n} GPU visible; peer bandwidth needs two"}))
        return 0
    out = {"gpus": n, "mib": args.mib, "unidirectional_GBs": {}}
    for i in range(n):
        for j in range(n):
            if i != j:
                out["unidirectional_GBs"][f"{i}->{j}"] = p2p_gbs(i, j, args.mib)
    vals = [v for v in out["unidirectional_GBs"].values() if v]
    out["min_GBs"], out["max_GBs"] = (min(vals), max(vals)) if vals else (None, None)
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
