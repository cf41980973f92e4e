"""Pages of an ncu report as text: from the .ncu-rep itself, or from the CSV exports
tools/profile_r02.sh writes on the GPU box (<prefix>_raw.csv[.gz], <prefix>_sass.csv[.gz])
so that the large report files need not travel back."""
import gzip
import os
import subprocess


def _read(path):
    if os.path.exists(path + ".gz"):
        with gzip.open(path + ".gz", "rt") as f:
            return f.read()
    with open(path) as f:
        return f.read()


def page(rep, which):
    """which: 'raw' or 'sass' (the source page with --print-source sass)."""
    if rep.endswith(".ncu-rep") and os.path.exists(rep):
        args = ["ncu", "-i", rep, "--page", "raw", "--csv"] if which == "raw" else \
               ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
        return subprocess.run(args, capture_output=True, text=True).stdout
    prefix = rep[:-len(".ncu-rep")] if rep.endswith(".ncu-rep") else rep
    return _read(f"{prefix}_{which}.csv")
