"""CLI invocations shared by the golden generator (reference CLI) and tests (device CLI)."""

import json
import os

CLI_MODELS = {
    "series": {"format": "rsr/1", "n_components": 3, "n_component_states": 2,
               "n_system_states": 2, "distribution": [[0.1, 0.9]] * 3,
               "system_function": {"name": "k_out_of_n", "k": 3}},
    "kofn3": {"format": "rsr/1", "n_components": 3, "n_component_states": 3,
              "n_system_states": 3, "distribution": [[0.2, 0.3, 0.5]] * 3,
              "system_function": {"name": "k_out_of_n", "k": 2}},
}
CLI_RUNS = [
    ["find-refs", "--model", "{series}", "--out-refs", "{out}", "--out-trace", "{trace}",
     "--samples", "2000", "--eps-u", "1e-3", "--seed", "5"],
    ["evaluate", "--model", "{series}", "--refs", "{refs}", "--out-report", "{out}",
     "--samples", "5000", "--seed", "5"],
    ["pmf", "--model", "{kofn3}", "--out", "{out}", "--samples", "5000", "--eps-u", "1e-3",
     "--seed", "2", "--parallel", "3"],
    ["oracle", "--model", "{series}", "--mode", "exact", "--out", "{out}"],
    ["oracle", "--model", "{kofn3}", "--mode", "exact", "--out", "{out}"],
    ["oracle", "--model", "{series}", "--mode", "mc", "--m-prime", "0", "--samples", "3000",
     "--seed", "9", "--out", "{out}"],
]


def strip_volatile(doc):
    """Drop timestamps / paths / elapsed fields that legitimately differ between runs."""
    if isinstance(doc, dict):
        return {k: strip_volatile(v) for k, v in doc.items()
                if k not in ("timestamp", "tool_version", "model_path", "refs_path")}
    if isinstance(doc, list):
        return [strip_volatile(v) for v in doc]
    return doc


def run_cli(main, workdir):
    """Run CLI_RUNS with the given main(); returns the JSON / trace outputs."""
    import csv
    paths = {}
    for name, doc in CLI_MODELS.items():
        p = os.path.join(workdir, f"{name}.json")
        with open(p, "w") as f:
            json.dump(doc, f)
        paths[name] = p
    outs = []
    refs_path = os.path.join(workdir, "out0.json")
    for i, argv in enumerate(CLI_RUNS):
        out = os.path.join(workdir, f"out{i}.json")
        trace = os.path.join(workdir, f"trace{i}.csv")
        args = [a.format(out=out, trace=trace, refs=refs_path, **paths) for a in argv]
        code = main(args)
        rec = {"code": code, "out": strip_volatile(json.load(open(out)))}
        if "--out-trace" in argv:
            with open(trace) as fh:
                rows = list(csv.reader(fh))
            rec["trace"] = [[r[0], r[2], r[3], r[4], r[5]] for r in rows]  # no elapsed / rss
        outs.append(rec)
    return outs
