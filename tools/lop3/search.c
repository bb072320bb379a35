/* Exhaustive search for minimum LOP3 networks (3-input boolean gates) computing a multi-output
 * lane function with don't-cares.  Used offline to derive the bitsliced formulas of the kernel
 * (the paper's own method, section 4, with LOP3 as the gate instead of 2-input AND/OR/XOR).
 *
 * Input (stdin): n_in n_out npoints, then per point: input_bits output_bits (unique target).
 * Wires are 64-bit truth tables over the 2^n_in assignments, restricted to the care mask.
 * A circuit = k intermediate gates (function enumerated) + one final gate per output whose
 * function is implied (the target must be consistent on the chosen 3 wires).  Outputs may
 * also be plain wires.  Prints every minimal solution found for the smallest k that works. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int NI, NO, NP;
static uint64_t care, target[4];
static uint64_t w[32];
static int nw;
static int gate_in[8][3], gate_fn[8];
static long long found = 0;
static int max_print = 20;

static uint64_t lop3(uint64_t a, uint64_t b, uint64_t c, int f) {
  uint64_t r = 0;
  for (int i = 0; i < 8; ++i)
    if ((f >> i) & 1) {
      uint64_t t = ((i & 4) ? a : ~a) & ((i & 2) ? b : ~b) & ((i & 1) ? c : ~c);
      r |= t;
    }
  return r;
}

/* is t a function of wires a,b,c on the care set?  returns the lop3 code or -1 */
static int implied(uint64_t t, uint64_t a, uint64_t b, uint64_t c) {
  int f = 0;
  for (int i = 0; i < 8; ++i) {
    uint64_t s = ((i & 4) ? a : ~a) & ((i & 2) ? b : ~b) & ((i & 1) ? c : ~c) & care;
    if (!s) continue;
    uint64_t on = t & s;
    if (on == s) f |= 1 << i;
    else if (on) return -1;
  }
  return f;
}

static int out_in[4][3], out_fn[4];

static int try_outputs(int k) {
  /* each output independently: a plain wire, or lop3 of 3 wires */
  for (int o = 0; o < NO; ++o) {
    int ok = 0;
    for (int a = 0; a < nw && !ok; ++a)
      if (((w[a] ^ target[o]) & care) == 0) { out_in[o][0] = a; out_in[o][1] = out_in[o][2] = -1; out_fn[o] = -1; ok = 1; }
    for (int a = 0; a < nw && !ok; ++a)
      for (int b = a + 1; b < nw && !ok; ++b)
        for (int c = b + 1; c < nw && !ok; ++c) {
          int f = implied(target[o], w[a], w[b], w[c]);
          if (f >= 0) { out_in[o][0] = a; out_in[o][1] = b; out_in[o][2] = c; out_fn[o] = f; ok = 1; }
        }
    if (!ok) return 0;
  }
  return 1;
}

static void print_solution(int k) {
  printf("solution: %d intermediate + outputs\n", k);
  for (int g = 0; g < k; ++g)
    printf("  w%d = lop3(w%d, w%d, w%d, 0x%02x)\n", NI + g, gate_in[g][0], gate_in[g][1], gate_in[g][2], gate_fn[g]);
  for (int o = 0; o < NO; ++o) {
    if (out_fn[o] < 0) printf("  out%d = w%d\n", o, out_in[o][0]);
    else printf("  out%d = lop3(w%d, w%d, w%d, 0x%02x)\n", o, out_in[o][0], out_in[o][1], out_in[o][2], out_fn[o]);
  }
  fflush(stdout);
}

static int count_final(void) {
  int n = 0;
  for (int o = 0; o < NO; ++o) n += out_fn[o] >= 0;
  return n;
}

static int best_total = 99;

static void rec(int g, int k) {
  if (g == k) {
    if (try_outputs(k)) {
      int total = k + count_final();
      if (total <= best_total) {
        best_total = total;
        if (found++ < max_print) { printf("total LOP3 = %d\n", total); print_solution(k); }
      }
    }
    return;
  }
  /* gate g takes inputs from wires < nw; canonical order: input triples increasing */
  for (int a = 0; a < nw; ++a)
    for (int b = a + 1; b < nw; ++b)
      for (int c = b + 1; c < nw; ++c) {
        for (int f = 1; f < 255; ++f) {
          /* independent consecutive gates commute: keep only the lexicographically ordered one */
          if (g > 0 && c < NI + g - 1) {
            const int* p = gate_in[g - 1];
            long long cur = ((long long)a << 24) | (b << 16) | (c << 8) | f;
            long long prv = ((long long)p[0] << 24) | (p[1] << 16) | (p[2] << 8) | gate_fn[g - 1];
            if (cur <= prv) continue;
          }
          uint64_t t = lop3(w[a], w[b], w[c], f) & care;
          int dup = 0;
          for (int i = 0; i < nw && !dup; ++i) if (((w[i] ^ t) & care) == 0 || ((~w[i] ^ t) & care) == 0) dup = 1;
          if (dup) continue;
          gate_in[g][0] = a; gate_in[g][1] = b; gate_in[g][2] = c; gate_fn[g] = f;
          w[nw++] = t;
          rec(g + 1, k);
          nw--;
        }
      }
}

int main(int argc, char** argv) {
  int kmax = argc > 1 ? atoi(argv[1]) : 2;
  if (scanf("%d %d %d", &NI, &NO, &NP) != 3) return 1;
  care = 0;
  for (int p = 0; p < NP; ++p) {
    int ib, ob;
    if (scanf("%d %d", &ib, &ob) != 2) return 1;
    care |= 1ull << ib;
    for (int o = 0; o < NO; ++o) if ((ob >> o) & 1) target[o] |= 1ull << ib;
  }
  for (int i = 0; i < NI; ++i) {
    uint64_t t = 0;
    for (int x = 0; x < (1 << NI); ++x) if ((x >> i) & 1) t |= 1ull << x;
    w[i] = t;
  }
  nw = NI;
  for (int k = 0; k <= kmax; ++k) {
    fprintf(stderr, "k = %d\n", k);
    rec(0, k);
    if (found) break;
  }
  if (!found) printf("no solution with <= %d intermediates\n", kmax);
  return 0;
}
