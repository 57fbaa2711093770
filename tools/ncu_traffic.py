"""Per-op-class DRAM traffic per launch from an ncu CSV with dram__bytes_{read,write}.sum
(+ gpu__time_duration.sum) over one timed bench round -> profiles/ncu_traffic.json."""
import collections
import csv
import json
import sys

NAME2OP = [("QuadConv1", "conv1_fwd"), ("HaloConv2<4, 0>", "conv2_fwd"), ("HaloConv2<4, 1>", "conv2_dgrad"),
           ("HaloConv2<4, false>", "conv2_fwd"), ("HaloConv2<(int)4, (bool)0>", "conv2_fwd"),
           ("HaloConv2<4, true>", "conv2_dgrad"), ("HaloConv2<(int)4, (bool)1>", "conv2_dgrad"),
           ("k_conv1_wgrad_q", "conv1_wgrad"), ("k_conv2_wgrad_halo", "conv2_wgrad"), ("k_head_cnn", "head"),
           ("Conv1Fwd", "conv1_fwd"), ("TcConv1Fwd", "conv1_fwd"), ("HaloConv2<", "conv2"), ("Conv2Fwd", "conv2_fwd"),
           ("Fc1Fwd", "fc1_fwd"), ("k_head", "head"), ("Fc1Dgrad", "fc1_dgrad"), ("Fc1Wgrad", "fc1_wgrad"),
           ("Conv2Dgrad", "conv2_dgrad"), ("Conv2Wgrad", "conv2_wgrad"), ("Conv1Wgrad", "conv1_wgrad"),
           ("k_reduce_conv1_tc", "conv1_reduce"), ("k_stage_x", "stage_x"), ("k_release_acc", "fedavg"),
           ("k_finalize", "fedavg"), ("k_admit", "admit"), ("MlpFc1Fwd", "mlp_fc1_fwd"),
           ("MlpFc1Wgrad", "mlp_fc1_wgrad"), ("RFwd", "resnet_fwd"), ("RDgrad", "resnet_dgrad"),
           ("RWgrad", "resnet_wgrad"), ("k_rhead", "resnet_head"), ("k_reduce_update", "reduce")]


def op_of(name):
    if "k_conv_halo" in name:
        return "conv2_dgrad" if "true" in name.split("k_conv_halo")[1][:20] else "conv2_fwd"
    for key, op in NAME2OP:
        if key in name:
            return op
    return name[:40]


def main(path, dtype, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        elif r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    # only the last round of the command (from its last admission on): the timed bench round
    ids = sorted(per, key=lambda x: int(x))
    last_admit = max((k for k, i in enumerate(ids) if "k_admit_params" in names[i]), default=0)
    for i in ids[last_admit:]:
        m = per[i]
        op = op_of(names[i])
        a = agg[op]
        a[0] += 1
        a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a[2] += m.get("gpu__time_duration.sum", 0)
    res = {}
    try:
        res = json.load(open(out))
    except Exception:
        pass
    for op, (n, b, t) in agg.items():
        res.setdefault(op, {})[dtype] = {"dram_bytes_per_launch": b / n, "launches": n,
                                         "ncu_ns_per_launch": t / n, "source": path}
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    for op, (n, b, t) in sorted(agg.items(), key=lambda x: -x[1][2]):
        print(f"{op:16s} n={n:5d} dram/launch={b / n / 1e6:9.2f} MB  ncu_time/launch={t / n / 1e3:8.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
