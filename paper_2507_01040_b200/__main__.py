"""`python -m paper_2507_01040_b200 serve` -- the JSON-lines layer server
(drop-in for `python -m mvkernels serve`, serve.py)."""
import sys

from .serve import serve_stdio

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "serve":
        sys.exit(serve_stdio())
    print("usage: python -m paper_2507_01040_b200 serve", file=sys.stderr)
    sys.exit(2)
