// ds_spec_builtin.cuh -- the stage types compiled into libds.so for K-N1s
// (ds_spec.cuh).  A stage type carries an Array-OL stage spec (ds_stage_spec,
// include/ds.h) as compile-time constants: pattern P, paving S, outputs Q,
// divisor D, bias B, origin O and the taps w(j, i).  Any other spec is
// compiled at run time from the same kernel source (ds_spec_jit.cu writes
// its stage types in this exact form).
#pragma once

namespace dss {

// SPEC's downscaler: hfilter_8to3 and vfilter_9to4
struct SpecH {
    static constexpr int P = 8, S = 8, Q = 3, D = 6, B = 3, O = 0;
    __host__ __device__ static constexpr int w(int j, int i) {
        constexpr int t[3][8] = {{1, 5, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 3, 3, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 5, 1}};
        return (j >= 0 && j < Q && i >= 0 && i < P) ? t[j][i] : 0;
    }
};
struct SpecV {
    static constexpr int P = 9, S = 9, Q = 4, D = 8, B = 4, O = 0;
    __host__ __device__ static constexpr int w(int j, int i) {
        constexpr int t[4][9] = {{3, 5, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 1, 7, 0, 0, 0, 0, 0},
                                 {0, 0, 0, 0, 0, 7, 1, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 5, 3}};
        return (j >= 0 && j < Q && i >= 0 && i < P) ? t[j][i] : 0;
    }
};

// The halo reading (bench.py --spec halo): 13-tap H and
// 14-tap V windows over the same 8 -> 3 / 9 -> 4 pavings, origins -2, so
// patterns overlap (halos) and wrap toroidally at the plane edges.
struct HaloH {
    static constexpr int P = 13, S = 8, Q = 3, D = 13, B = 6, O = -2;
    __host__ __device__ static constexpr int w(int j, int i) {
        constexpr int t[3][13] = {{1, 3, 5, 3, 1, 0, 0, 0, 0, 0, 0, 0, 0},
                                  {0, 0, 0, 1, 3, 5, 3, 1, 0, 0, 0, 0, 0},
                                  {0, 0, 0, 0, 0, 0, 1, 3, 5, 3, 1, 0, 0}};
        return (j >= 0 && j < Q && i >= 0 && i < P) ? t[j][i] : 0;
    }
};
struct HaloV {
    static constexpr int P = 14, S = 9, Q = 4, D = 10, B = 5, O = -2;
    __host__ __device__ static constexpr int w(int j, int i) {
        constexpr int t[4][14] = {{1, 2, 4, 2, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0},
                                  {0, 0, 1, 2, 4, 2, 1, 0, 0, 0, 0, 0, 0, 0},
                                  {0, 0, 0, 0, 0, 1, 2, 4, 2, 1, 0, 0, 0, 0},
                                  {0, 0, 0, 0, 0, 0, 0, 0, 1, 2, 4, 2, 1, 0}};
        return (j >= 0 && j < Q && i >= 0 && i < P) ? t[j][i] : 0;
    }
};

}  // namespace dss
