"""Constants of the register-file plan records (csrc/rf_plan.h), for host-side models."""


class RF:
    NONE = 0xFFFFFFFF
    WAIT_FILL = 0x80000000
    STORE_SPILL = 0x80000000
    RING = 16
    SB_LNEG, SB_RNEG, SB_STORE, SB_DEST_STORED, SB_HAZARD, SB_DEST_FIRST = 1, 2, 4, 8, 16, 32
    SB_REUSE_L, SB_REUSE_R = 64, 128
    FF_FIRST = 1
