"""Build an experimental copy of libusp.so from a patched copy of csrc/.

    python tools/build_variant.py OUT_DIR [--define NAME[=VAL] ...] [--patch FILE:OLD_FILE_SNIPPET_FILE:NEW_SNIPPET_FILE]

Copies paper_2207_14222_b200/csrc to OUT_DIR/csrc, applies -D defines, and
builds OUT_DIR/libusp.so with the same nvcc flags as the product build
(for in-process A/B runs with tools/gpu/kab.py).  The product library is
not touched.
"""
import argparse
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--from-git", default=None, help="take csrc/ from this git revision instead of the tree")
    args = ap.parse_args()
    from paper_2207_14222_b200 import build as B

    out = os.path.abspath(args.out)
    csrc = os.path.join(out, "csrc")
    shutil.rmtree(out, ignore_errors=True)
    os.makedirs(out)
    if args.from_git:
        import subprocess
        import tarfile
        import io

        tar = subprocess.run(["git", "-C", ROOT, "archive", args.from_git, "paper_2207_14222_b200/csrc"],
                             capture_output=True, check=True).stdout
        tarfile.open(fileobj=io.BytesIO(tar)).extractall(out)
        shutil.move(os.path.join(out, "paper_2207_14222_b200", "csrc"), csrc)
    else:
        shutil.copytree(B.CSRC, csrc)
    B.CSRC = csrc
    B.BUILD = os.path.join(out, "_build")
    B.LIB = os.path.join(out, "libusp.so")
    B.FLAGS = B.FLAGS + [f"-D{d}" for d in args.define]
    B.FLAGS = [f if f != os.path.join(ROOT, "paper_2207_14222_b200", "csrc") else csrc for f in B.FLAGS]
    print(B.build(force=True))


if __name__ == "__main__":
    main()
