"""Helpers shared by the tests (unique module name: `tests` clashes on sys.path)."""


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
