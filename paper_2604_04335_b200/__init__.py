"""GenServe DiT-step hot path on B200 (sm_100a): thin Python binding over libgs.so."""
