"""B200 analogue of the paper's Table 1 + the reference's accuracy experiments.

    python scripts/table1.py [out.md]

Runs paper_1401_0248_b200.harness on cuda:0 and writes a markdown report
(Gelem/s, paper convention of one add per element).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import harness as H  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/table1.md"
    torch.cuda.set_device(0)
    rows = H.table1()
    lines = ["# Table 1 on B200 (Gelem/s; paper convention: one add per element)", "",
             f"device: {torch.cuda.get_device_name(0)}; tiers: small 256 KiB, medium 32 MiB (L2-resident, "
             "no flush: the paper's 'medium fits L3'), large 2 GiB per operand (HBM); noread = recurrence on "
             "register-resident addends (p-rows); read1/read2 = direct sum/dot.", "",
             H.format_table1(rows), ""]
    acc = H.run_accuracy_table()
    lines += ["## accuracy table (accuracy.run_accuracy_table, n=1e6, seed 1, cuda flavor)", "",
              "| precision | generator | interval | method | rel_error |", "|---|---|---|---|---|"]
    lines += [f"| {r.precision} | {r.generator} | {r.interval} | {r.method} | {r.rel_error:.3e} |" for r in acc]
    for fl in (tfb.Flavor.sequential(), tfb.Flavor.cuda()):
        hrs = H.run_hours100(fl)
        lines += ["", f"## 100-hours test, flavor {fl}", "", "| method | hours | deviation | estimate |",
                  "|---|---|---|---|"]
        lines += [f"| {r.method} | {r.result_hours:.6f} | {r.deviation_hours:.3e} | "
                  f"{'' if r.estimate_hours is None else f'{r.estimate_hours:.6f}'} |" for r in hrs]
    pts, slopes = H.run_scaling_study(trials=20)
    lines += ["", "## scaling study (median |rel err|, 20 trials, f32 NR, cuda flavor)", "",
              "| n | method | median |rel err| |", "|---|---|---|"]
    lines += [f"| {n} | {m} | {e:.3e} |" for n, m, e in pts]
    lines += ["", f"fitted log-log slopes: {json.dumps(slopes)}"]
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    with open(out.replace(".md", ".json"), "w") as f:
        json.dump([r.__dict__ for r in rows], f)


if __name__ == "__main__":
    main()
