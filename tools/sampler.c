// sampler.c — a tiny in-process sampling profiler for the host side of the
// eager step (LD_PRELOAD; no perf on the GPU boxes).
//
//   gcc -O2 -shared -fPIC -o tools/libsampler.so tools/sampler.c -ldl -lrt
//   SAMPLER_OUT=gpurun_out/samples.txt LD_PRELOAD=tools/libsampler.so python tools/host_profile.py c4
//
// SIGPROF every SAMPLER_US (default 200) µs of process CPU time; each sample
// stores the first SAMPLER_DEPTH return addresses of the interrupted thread.
// Sampling is armed/disarmed by the program through sampler_arm(int) (dlsym),
// or for the whole run when SAMPLER_ALWAYS=1.  At exit the samples are
// written as "count module+offset;module+offset;..." lines (innermost first),
// resolved here with addr2line (tools/sampler_report.py).
#define _GNU_SOURCE
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/time.h>
#include <time.h>

#define MAXS 100000
#define MAXD 40
static void* g_st[MAXS][MAXD];
static int g_n[MAXS];
static volatile int g_cnt = 0;
static volatile int g_armed = 0;
static int g_depth = 32;

static void on_prof(int sig, siginfo_t* si, void* uc) {
  (void)sig; (void)si; (void)uc;
  if (!g_armed) return;
  int i = __sync_fetch_and_add(&g_cnt, 1);
  if (i >= MAXS) return;
  void* buf[MAXD + 2];
  int n = backtrace(buf, g_depth + 2);
  // drop this handler's own frame and the signal trampoline
  int k = 0;
  for (int j = 2; j < n && k < g_depth; ++j) g_st[i][k++] = buf[j];
  g_n[i] = k;
}

void sampler_arm(int on) { g_armed = on; }

static void dump(void) {
  const char* out = getenv("SAMPLER_OUT");
  if (!out) return;
  g_armed = 0;
  FILE* f = fopen(out, "w");
  if (!f) return;
  int n = g_cnt < MAXS ? g_cnt : MAXS;
  fprintf(f, "# samples %d interval_us %s\n", n, getenv("SAMPLER_US") ? getenv("SAMPLER_US") : "200");
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < g_n[i]; ++k) {
      Dl_info d;
      if (dladdr(g_st[i][k], &d) && d.dli_fname)
        fprintf(f, "%s%s+0x%lx", k ? ";" : "", d.dli_fname,
                (unsigned long)((uintptr_t)g_st[i][k] - (uintptr_t)d.dli_fbase - 1));
      else
        fprintf(f, "%s?+0x%lx", k ? ";" : "", (unsigned long)(uintptr_t)g_st[i][k]);
    }
    fputc('\n', f);
  }
  fclose(f);
}

__attribute__((constructor)) static void init(void) {
  if (!getenv("SAMPLER_OUT")) return;
  const char* d = getenv("SAMPLER_DEPTH");
  if (d) g_depth = atoi(d) > MAXD ? MAXD : atoi(d);
  void* warm[4];
  backtrace(warm, 4);  // load libgcc's unwinder outside the handler
  struct sigaction sa;
  memset(&sa, 0, sizeof(sa));
  sa.sa_sigaction = on_prof;
  sa.sa_flags = SA_SIGINFO | SA_RESTART;
  sigaction(SIGPROF, &sa, NULL);
  // a POSIX CPU-time timer (hrtimer based; setitimer's ITIMER_PROF ticks at
  // the scheduler HZ, i.e. 4 ms resolution)
  const char* us = getenv("SAMPLER_US");
  long u = us ? atol(us) : 200;
  timer_t tid;
  struct sigevent sev;
  memset(&sev, 0, sizeof(sev));
  sev.sigev_notify = SIGEV_SIGNAL;
  sev.sigev_signo = SIGPROF;
  if (timer_create(CLOCK_PROCESS_CPUTIME_ID, &sev, &tid) == 0) {
    struct itimerspec its = {{0, u * 1000}, {0, u * 1000}};
    timer_settime(tid, 0, &its, NULL);
  }
  if (getenv("SAMPLER_ALWAYS")) g_armed = 1;
  atexit(dump);
}
