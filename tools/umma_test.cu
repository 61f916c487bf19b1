// Standalone check of the tcgen05 kind::i8 seed contraction (seed_umma.cuh) against a CPU
// reference: nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2503_17911_b200/csrc
//            tools/umma_test.cu -o /tmp/umma_test && /tmp/umma_test
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2503_17911_b200/csrc/seed.cu"

int run(int nq, int S, int cbp, unsigned seed, bool ip = false, bool sq4 = false) {
    // SQ4: A = the operand (2 * cbp bytes per query, nibble-plane order), B = packed codes
    const int ka = sq4 ? 2 * cbp : cbp;
    std::vector<uint8_t> hq((size_t)nq * ka), hs((size_t)S * cbp);
    srand(seed);
    for (auto &v : hq) v = sq4 && !ip ? (rand() & 15) : (rand() & 255);
    for (auto &v : hs) v = rand() & 255;
    uint8_t *dq, *ds;
    int32_t *dt;
    cudaMalloc(&dq, hq.size());
    cudaMalloc(&ds, hs.size());
    cudaMalloc(&dt, (size_t)nq * S * 4);
    int *derr;
    cudaMalloc(&derr, 4);
    cudaMemset(derr, 0, 4);
    cudaMemcpy(dq, hq.data(), hq.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs.data(), hs.size(), cudaMemcpyHostToDevice);
    cudaMemset(dt, 0xff, (size_t)nq * S * 4);
    uint8_t *dso;
    cudaMalloc(&dso, vsag::seed_operand_bytes(S, cbp, sq4 ? 4 : 8));
    vsag::launch_seed_operand(ds, S, cbp, sq4 ? 4 : 8, dso, 0);
    cudaError_t le = vsag::launch_seed_tau_umma(dq, nq, dso, S, ka, ip, dt, derr, 0);
    if (le != cudaSuccess) {
        printf("launch error %s\n", cudaGetErrorString(le));
        return 1;
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<int32_t> ht((size_t)nq * S);
    cudaMemcpy(ht.data(), dt, ht.size() * 4, cudaMemcpyDeviceToHost);
    long long bad = 0, shown = 0;
    for (int q = 0; q < nq; q++)
        for (int s = 0; s < S; s++) {
            int ref = 0;
            for (int k = 0; k < ka; k++) {
                int cv;  // the code value at operand position k
                if (sq4) {  // position k: code word k / 8, plane (k / 4) % 2, byte k % 4
                    const int w = k / 8, plane = (k / 4) % 2, t = k % 4;
                    const uint8_t byte = hs[(size_t)s * cbp + 4 * w + t];
                    cv = plane ? byte >> 4 : byte & 15;
                } else {
                    cv = hs[(size_t)s * cbp + k];
                }
                if (ip) {  // int8 weights x codes, tau = -dot
                    ref -= (int)(int8_t)hq[(size_t)q * ka + k] * cv;
                } else {
                    int d = (int)hq[(size_t)q * ka + k] - cv;
                    ref += d * d;
                }
            }
            if (ht[(size_t)q * S + s] != ref) {
                if (shown++ < 5) printf("  q %d s %d got %d want %d\n", q, s, ht[(size_t)q * S + s], ref);
                bad++;
            }
        }
    printf("%s%s nq %d S %d cbp %d: %lld mismatches\n", ip ? "ip" : "l2", sq4 ? "/sq4" : "", nq, S, cbp, bad);
    cudaFree(dq);
    cudaFree(ds);
    cudaFree(dt);
    cudaFree(dso);
    int herr = 0;
    cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost);
    if (herr) printf("  timeout flag set\n");
    return bad != 0 || herr != 0;
}

int main() {
    int fails = 0;
    fails += run(128, 256, 128, 1);
    fails += run(300, 1000, 128, 2);
    fails += run(257, 513, 192, 3);
    fails += run(50, 100, 16, 4);
    fails += run(300, 1000, 128, 5, true);
    fails += run(130, 300, 768, 6, true);
    fails += run(300, 700, 64, 7, false, true);   // C4-like: 64-byte codes, K 128
    fails += run(100, 600, 480, 8, false, true);  // C2-like: K 960 (7.5 blocks)
    fails += run(90, 260, 48, 9, true, true);     // IP SQ4, partial K block
    fails += run(3000, 1024, 128, 10);            // C1 shape
    fails += run(130, 16384, 480, 11, false, true);   // C2 shape (S = 16384, K 960)
    fails += run(333, 256, 768, 12, true);        // C3 shape (IP, K 768)
    printf(fails ? "FAIL\n" : "ALL OK\n");
    return fails;
}
