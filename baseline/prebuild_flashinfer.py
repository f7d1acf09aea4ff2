"""Prebuild (cross-compile for sm_100a) the FlashInfer module the FP16
full-KV baseline uses, into baseline/flashinfer_ws (travels to the GPU box;
git-ignored). bench.py points FLASHINFER_WORKSPACE_BASE there so a fresh box
does not spend minutes in FlashInfer's JIT. Library code, used only for the
baseline arm of the comparison."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("FLASHINFER_WORKSPACE_BASE", os.path.join(HERE, "flashinfer_ws"))
os.environ.setdefault("FLASHINFER_CUDA_ARCH_LIST", "10.0a")

import torch  # noqa: E402
from flashinfer.prefill import get_batch_prefill_module  # noqa: E402


def main():
    mod = get_batch_prefill_module("fa2", torch.float16, torch.float16, torch.float16, torch.int32,
                                   128, 128, 0, False, False, False)
    print("built", mod)


if __name__ == "__main__":
    sys.exit(main())
