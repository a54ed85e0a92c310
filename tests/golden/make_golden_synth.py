"""SHA-256 digests of the reference's synthetic CIFAR corpora (data.py:114-165)
for the three block styles, for tests/test_host.py::test_synth_styles_match_reference.
Run here with the reference importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_synth.py
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from qtape import data as D  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [(5, 300, 96.0, "sparse"), (5, 300, 64.0, "natural"), (3, 200, 32.0, "smooth")]


def main():
    out = []
    for seed, n, noise, style in CASES:
        images, labels = D.synth_cifar_like(seed, n, noise=noise, style=style)
        h = hashlib.sha256(images.tobytes() + labels.astype("int64").tobytes()).hexdigest()
        out.append({"seed": seed, "n": n, "noise": noise, "style": style, "sha256": h})
    with open(os.path.join(HERE, "synth_styles.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out)


if __name__ == "__main__":
    main()
