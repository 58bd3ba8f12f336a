"""Named random substreams (restates reference ``streams.py:16-36``).

A stream is addressed by (seed, *path); string path components map to
integers with CRC-32 (``streams.py:33-36``) and become the SeedSequence
spawn key feeding a Philox bit generator (``streams.py:29-30``).
"""

import zlib

import numpy as np


def _key(part):
    # streams.py:33-36: ints pass through, everything else is CRC-32 of str()
    if isinstance(part, (int, np.integer)):
        return int(part)
    return zlib.crc32(str(part).encode())


def substream(seed, *path):
    """numpy Generator for the named substream (streams.py:16-30)."""
    seq = np.random.SeedSequence(entropy=seed,
                                 spawn_key=tuple(_key(p) for p in path))
    return np.random.Generator(np.random.Philox(seq))
