// fftw3.h stand-in for building the reference sources verbatim (oracle/_ref, test
// infrastructure). Declares the FFTW3 calls proj/src/fft.cpp makes (fft.cpp:32-58); the
// definitions (ref_shim/fftw_shim.cpp) are an own radix-2 transform with FFTW's
// conventions: FFTW_FORWARD = -1 gives X_k = sum_j x_j e^{-2 pi i jk/n}, FFTW_BACKWARD
// = +1 the unnormalised inverse. FFTW itself (unpinned, absent here) chooses its own
// codelets, so its results agree with these to rounding, not bit for bit.
#pragma once
typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;
#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
fftw_complex* fftw_alloc_complex(unsigned long n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
