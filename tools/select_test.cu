// Standalone check of seed selection (select.cu) against a CPU reference: top-L (tau, id) of S.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -I paper_2503_17911_b200/csrc \
//      tools/select_test.cu -o /tmp/select_test && /tmp/select_test
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2503_17911_b200/csrc/select.cu"

int run(int nq, int S, int L, int range, unsigned seed) {
    std::vector<int32_t> tau((size_t)nq * S), entry(S);
    srand(seed);
    for (auto &v : tau) v = (rand() % range) - (range / 3);
    for (int i = 0; i < S; i++) entry[i] = 3 * i + 1;
    int32_t *dt, *de, *dp;
    uint64_t *dk;
    cudaMalloc(&dt, tau.size() * 4);
    cudaMalloc(&de, S * 4);
    cudaMalloc(&dk, (size_t)nq * L * 8);
    cudaMalloc(&dp, nq * 4);
    cudaMemcpy(dt, tau.data(), tau.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(de, entry.data(), S * 4, cudaMemcpyHostToDevice);
    cudaMemset(dk, 0xee, (size_t)nq * L * 8);
    vsag::launch_seed_select(dt, de, S, nq, L, dk, dp, 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<uint64_t> hk((size_t)nq * L);
    std::vector<int> hp(nq);
    cudaMemcpy(hk.data(), dk, hk.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hp.data(), dp, nq * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    const int need = std::min(L, S);
    for (int q = 0; q < nq; q++) {
        std::vector<std::pair<int, int>> ref(S);
        for (int i = 0; i < S; i++) ref[i] = {tau[(size_t)q * S + i], entry[i]};
        std::sort(ref.begin(), ref.end());
        bool ok = hp[q] == need;
        for (int t = 0; t < need && ok; t++) {
            const uint64_t k = hk[(size_t)q * L + t];
            const int tv = (int)((uint32_t)(k >> 32) ^ 0x80000000u), id = (int)((uint32_t)k >> 1);
            if (tv != ref[t].first || id != ref[t].second) {
                if (bad < 5) printf("  q %d t %d got (%d, %d) want (%d, %d)\n", q, t, tv, id, ref[t].first, ref[t].second);
                ok = false;
            }
        }
        bad += !ok;
    }
    printf("nq %d S %d L %d range %d: %ld bad queries\n", nq, S, L, range, bad);
    cudaFree(dt); cudaFree(de); cudaFree(dk); cudaFree(dp);
    return bad != 0;
}

int main() {
    int f = 0;
    f += run(100, 128, 64, 1000000, 1);
    f += run(100, 128, 64, 50, 2);
    f += run(300, 1024, 130, 8000000, 3);
    f += run(300, 1000, 200, 100, 4);
    f += run(300, 256, 256, 1 << 30, 5);
    f += run(300, 37, 10, 1000, 6);
    f += run(300, 512, 100, 1 << 30, 7);
    f += run(300, 2000, 100, 1000000, 8);
    printf(f ? "FAIL\n" : "ALL OK\n");
    return f;
}
