"""ezLDA (arXiv 2007.08725) three-branch Gibbs hot path, B200-native (sm_100a).

The compute path lives in libezlda.so (csrc/, C ABI declared in include/ezlda.h);
`paper_2007_08725_b200.lda` is the thin ctypes binding.  Importing this package
does not load the shared library; `lda.load()` does, and raises if it is missing.
"""
__all__ = ["lda", "synth"]
