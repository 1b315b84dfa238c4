// Constants of the processors (mg/processors.py:19-39) and device tables.
#pragma once
#include <cuda_runtime.h>

#define MGB_EQ_LEN 2047
#define MGB_EQ_BINS 1024
#define MGB_REV_NFFT 384
#define MGB_REV_HOP 192
#define MGB_REV_PBINS 192
#define MGB_REV_BINS 193
#define MGB_REV_FRAMES 313
#define MGB_REV_LEN 60000
#define MGB_ENV_LEN 8192
#define MGB_ENV_EPS 1e-8
#define MGB_DLY_TAPS 20
#define MGB_DLY_WIN 3000
#define MGB_COLOR_LEN 39
#define MGB_COLOR_BINS 20
#define MGB_DLY_FIR (MGB_DLY_TAPS * MGB_DLY_WIN + MGB_COLOR_LEN - 1)
#define MGB_GS_EPS 1e-8

extern __device__ float2 g_rev_spec[2][MGB_REV_FRAMES][MGB_REV_BINS];
extern __device__ float g_rev_inv_wss[MGB_REV_LEN];
extern __device__ double g_hann2047[MGB_EQ_LEN];
extern __device__ double g_cos39[MGB_COLOR_LEN], g_hann39[MGB_COLOR_LEN];
