#!/usr/bin/env python3
"""Regenerates the committed golden fixtures from the REFERENCE compiler.

Test infrastructure only.  Requires oracle/_ref/ (built by `make -C oracle/ref_harness`
from the read-only reference headers under /root/reference/proj/include).

Writes:
  tests/golden/ir/<name>.ir.json          fused IR, reference schedule() + serialize()
  tests/golden/ir/<name>.unfused.ir.json  same program without fuse()  (fusion-equivalence tests)
  tests/golden/ir/<name>.ll.ir.json       protocol "ll" variants of the C4 configs
  tests/golden/symbolic/<name>.json       reference symbolic end state (core.hpp chunk algebra) +
                                          postcondition verdict (chunk_dag.hpp:133-149)
  tests/golden/MANIFEST.json              sha256 of every IR; the 17 SURVEY.md Appendix D digests
                                          are asserted here (and re-checked by tests/test_golden.py)
"""
import ctypes
import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(REPO, "oracle", "_ref")

# SHA-256 of the fused IRs written by the reference serialize().
SURVEY_DIGESTS = {
    "allpairs_ar_2": "f7d9e230f6a26afb3c268f26ec100111a2b295b220326a35b4fd1d6142eaf42d",
    "allpairs_ar_4": "38c7b50943889d26270ccc05cfba4d6da17bed3eb4bdeb3340a1f2b529f47feb",
    "allpairs_ar_8": "41629d8e7cb123ac7299d4e885568d2d1d61489698d77a5dff0422291f4f931d",
    "hier_ar_2x4_par1": "53a4fdcc16c7241f5db9b1c0c61a69ecb64a58ae9f8aba1ace6fa2bf546fe653",
    "hier_ar_2x4_par2": "5e2dd2cd0a264fa19a36fe822aa962464020a2fc32e994e895ef40f94d009880",
    "ring_ag_2": "462c9cbe240cd43fe25c83536739f3a6186441bf6b5b5ae8bbfb05d56b5cb313",
    "ring_ag_4": "98c17baaba0b9783079f1ef46e8b1e1b6184e725c68fb55fa5ade3afc8b6da54",
    "ring_ag_8": "377409d197a6e4ac360af21d0269aa36b3e8d9c500de289f1ff63f24a3cc9a39",
    "ring_ar_8_ch1": "f21f712735665ef8790f58358c79060f0591e16bd23ce7328c10616ad90758b4",
    "ring_ar_8_ch8_inst1": "fb60efae14cb415a725c481e892e0100c43c7e7602d51c6a86d425c59ce87aa9",
    "ring_ar_8_ch8_inst4": "4ddb6ac066da16db0f9470d30d6eef48a4d8b3ae57fbb84144e73c05cf9fd4df",
    "ring_ar_8_inst4_auto": "51546694bc1883c452ac3d65c045303e0ab05dcb599f0c443264ec6677a6db6d",
    "ring_rs_2": "83bf93534cf7239c27061cecaa63b26c7aea5cb1c2d0f94644652971fc4ee1e9",
    "ring_rs_4": "587dd54799ec1b9ad7ffaaa9ae69df8065c2ede06f3fb7ee95cc26d2c6ebaf8c",
    "ring_rs_8": "419ce284fc74a5fd77fc80c3848110dd52934b81e68cd855b8d4cf85b922e491",
    "twostep_a2a_1x8": "954e301719da86409285045debfe6aa88208285ce5a86b77b87103c699784307",
    "twostep_a2a_2x4": "2e0e5b8e5d303b36117ac07291633bf3d6668b9145f253c61e17b8d3c41e2b3a",
}

LL_VARIANTS = ["ring_ar_8_ch8_inst4", "ring_ar_8_ch1", "ring_ar_8_inst4_auto", "twostep_a2a_1x8"]


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def main():
    tool = os.path.join(REF, "ref_tool")
    lib = ctypes.CDLL(os.path.join(REF, "libref.so"))
    lib.ref_compile.restype = ctypes.c_void_p
    lib.ref_symbolic.restype = ctypes.c_void_p
    lib.ref_free.argtypes = [ctypes.c_void_p]

    def take(p):
        s = ctypes.string_at(p).decode()
        lib.ref_free(p)
        return s

    irdir = os.path.join(HERE, "ir")
    symdir = os.path.join(HERE, "symbolic")
    os.makedirs(irdir, exist_ok=True)
    os.makedirs(symdir, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.check_call([tool, "gen", tmp])
        for f in sorted(os.listdir(tmp)):
            with open(os.path.join(tmp, f), "rb") as src, open(os.path.join(irdir, f), "wb") as dst:
                dst.write(src.read())
    for name in LL_VARIANTS:
        text = take(lib.ref_compile(name.encode(), 1, 1))
        assert not text.startswith("ERROR"), text
        with open(os.path.join(irdir, name + ".ll.ir.json"), "w") as f:
            f.write(text)

    manifest = {}
    for f in sorted(os.listdir(irdir)):
        if not f.endswith(".ir.json"):
            continue
        manifest[f] = sha(os.path.join(irdir, f))
        with open(os.path.join(irdir, f)) as fh:
            text = fh.read()
        sym = json.loads(take(lib.ref_symbolic(text.encode())))
        assert sym["passed"], (f, sym["error"])
        with open(os.path.join(symdir, f.replace(".ir.json", ".json")), "w") as fh:
            json.dump(sym, fh, sort_keys=True)
    for name, digest in SURVEY_DIGESTS.items():
        got = manifest[name + ".ir.json"]
        if got != digest:
            sys.exit(f"fixture {name}: sha256 {got} != SURVEY.md Appendix D {digest}")
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump({"survey_digests": SURVEY_DIGESTS, "sha256": manifest}, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"{len(manifest)} fixtures, {len(SURVEY_DIGESTS)} SURVEY digests reproduced")


if __name__ == "__main__":
    main()
