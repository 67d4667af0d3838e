"""Effective key set of the multi-shot attention sink (TEST INFRASTRUCTURE).

PAPER.md:187 (§4.2): sliding-window self-attention with KV caching caps the
per-step work at O(W * L_c).  PAPER.md:246-249 (§4.2): the global sink A_g is
the first S_g frames; the shot-level sink A_s is tracked by two scalar
pointers (start, len); at chunk step t the effective set is
``K_eff(t) = A_g ∪ A_s ∪ KV_[t-W, t)`` with overlapping tokens deduplicated.
PAPER.md:45: the current chunk attends to its own tokens (bidirectional).

Readings: Z9 the current chunk is attended from the cache;
Z10 ``window_frames`` counts frames *including* the current chunk; Z11 sinks
are counted in frames and ranges are token-exact.

All quantities here are logical (frame / token) indices, not cache slots.
"""
from __future__ import annotations


def key_frames(chunk_index, frames_per_chunk, sink_frames, window_frames,
               shot_start_frame=0, shot_len_frames=0):
    """Sorted list of the distinct frames in K_eff(t) for chunk t = chunk_index."""
    t, fc = int(chunk_index), int(frames_per_chunk)
    f_end = (t + 1) * fc                                   # one past the current chunk's last frame
    frames = set()
    frames.update(range(0, min(int(sink_frames), f_end)))                     # A_g
    s0, sl = int(shot_start_frame), int(shot_len_frames)
    frames.update(f for f in range(s0, s0 + sl) if 0 <= f < f_end)           # A_s
    frames.update(range(max(0, f_end - int(window_frames)), f_end))           # KV_[t-W, t)
    frames.update(range(f_end - fc, f_end))                                   # current chunk
    return sorted(frames)


def key_token_ranges(chunk_index, frames_per_chunk, tokens_per_frame, sink_frames,
                     window_frames, shot_start_frame=0, shot_len_frames=0):
    """K_eff(t) as ascending, disjoint, non-adjacent half-open token ranges [(a, b), ...]."""
    frames = key_frames(chunk_index, frames_per_chunk, sink_frames, window_frames,
                        shot_start_frame, shot_len_frames)
    ranges = []
    for f in frames:
        a, b = f * tokens_per_frame, (f + 1) * tokens_per_frame
        if ranges and ranges[-1][1] == a:
            ranges[-1] = (ranges[-1][0], b)
        else:
            ranges.append((a, b))
    return ranges


def key_tokens(*args, **kw):
    """Flat ascending list of logical key token indices (for brute-force checks)."""
    out = []
    for a, b in key_token_ranges(*args, **kw):
        out.extend(range(a, b))
    return out
