"""python -m paper_1205_1098_b200 search KERNEL [--strategy ...] [--fitness analytic|gpu] ...

The one command the hot path needs from the reference's CLI: `matfuse search --fitness`
(cli.py:205-246) over the GPU launch variants.  Everything else the reference's CLI does
(parse / enumerate / corpus tables) is compile-time tooling and out of scope."""
import sys

from .search import EXIT_USAGE, main as search_main


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv or argv[0] != "search":
        print(__doc__, file=sys.stderr)
        return EXIT_USAGE
    return search_main(argv[1:])


if __name__ == "__main__":
    raise SystemExit(main())
