"""gram_traffic.json from an ncu metrics launch list of one C5 step.

Input: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
       -k regex:"gram_tf32_2cta|gram2_reduce" --csv (profiles/gpu_round.sh part `traffic`).
The mode-1 Gram is every gram_tf32_2cta_kernel K-launch before the first
gram2_reduce (64 at the default 1024 K-blocks per unit and launch) plus that reduce: bench.py's roofline treats that
logical Gram (I^2 J flops) as one launch, so its traffic is their sum."""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def main(src, dst, n_gram=0):
    rows, hdr = [], None
    for r in csv.reader(open(src)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rows.append(dict(zip(hdr, r)))
    launches = {}
    for d in rows:
        key = (d["ID"], d["Kernel Name"])
        launches.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT.get(
            d["Metric Unit"], 1)
    order = sorted(launches, key=lambda k: int(k[0]))
    # the mode-1 Gram = every K-launch before the first reduction (n_gram <= 0), or the first n_gram
    first_red = next(i for i, k in enumerate(order) if "gram2_reduce" in k[1])
    gram = [launches[k] for k in order[:first_red] if "gram_tf32_2cta" in k[1]]
    if n_gram > 0:
        gram = gram[:n_gram]
    red = [launches[order[first_red]]]
    sel = gram + red
    rd = sum(x["dram__bytes_read.sum"] for x in sel)
    wr = sum(x["dram__bytes_write.sum"] for x in sel)
    out = {"kernel": "gram_tf32_2cta_kernel x%d K-launches + gram2_reduce" % len(gram),
           "config": "C5 mode 1 (n=0), 2048^3 f32", "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_launch": rd + wr, "algorithmic_bytes": 4.0 * 2048 ** 3,
           "ncu_time_s": sum(x["gpu__time_duration.sum"] for x in sel), "source": src}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/gram_traffic.json",
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
