// synth_host.cpp — host side of the seekable synthetic generator (psattn_synth.h).
#include <cmath>
#include <vector>

#include "psattn_synth.h"
#include "synth.h"

extern "C" {

void psattn_synth_direction(const psattn_synth_params* p, int64_t unit_id, float* out) {
    psa_synth::direction(p->seed, unit_id, p->dim, out);
}

void psattn_synth_query(const psattn_synth_params* p, int64_t unit_id, int32_t head, float* out) {
    const int d = p->dim;
    std::vector<float> dir(d), g(d);
    psa_synth::direction(p->seed, unit_id, d, dir.data());
    // per-head perturbation: a unit vector from its own stream (unit*64 + head)
    psa_synth::direction(p->seed ^ 0x51ED270B27F1A3C5ULL, unit_id * 64 + head, d, g.data());
    std::vector<double> v(d);
    double ss = 0.0;
    for (int i = 0; i < d; ++i) {
        v[i] = (double)dir[i] + 0.1 * (double)g[i];
        ss += v[i] * v[i];
    }
    const double s = std::sqrt((double)d) / std::sqrt(ss);
    for (int i = 0; i < d; ++i) out[i] = (float)(v[i] * s);
}

int psattn_synth_is_planted(const psattn_synth_params* p, int64_t unit_id, int64_t block) {
    return psa_synth::is_planted(p->seed, p->planted_prob, unit_id, block);
}

void psattn_synth_unit_host(const psattn_synth_params* p, int64_t unit_id, int64_t first_block, int64_t n_blocks,
                            int64_t n_tokens_total, float* keys, float* values) {
    const int d = p->dim, T = p->block_tokens;
    std::vector<float> dir(d);
    psa_synth::direction(p->seed, unit_id, d, dir.data());
    for (int64_t bi = 0; bi < n_blocks; ++bi) {
        const int64_t b = first_block + bi;
        const int planted = psa_synth::is_planted(p->seed, p->planted_prob, unit_id, b);
        for (int t = 0; t < T; ++t) {
            const int64_t tok = b * T + t;
            for (int i = 0; i < d; ++i) {
                const size_t idx = ((size_t)bi * T + t) * d + i;
                float kx = 0.0f, vx = 0.0f;
                if (tok < n_tokens_total) {
                    kx = psa_synth::key_at(p->seed, unit_id, tok, i, d, planted, p->skew, dir[i]);
                    vx = psa_synth::value_at(p->seed, unit_id, b, tok, i, d);
                    if (p->round_bf16) {
                        kx = psa_synth::round_bf16(kx);
                        vx = psa_synth::round_bf16(vx);
                    }
                }
                keys[idx] = kx;
                values[idx] = vx;
            }
        }
    }
}

}  // extern "C"
