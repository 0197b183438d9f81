#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <time.h>
#include <stdint.h>
static double now(){struct timespec t;clock_gettime(CLOCK_MONOTONIC,&t);return t.tv_sec*1e3+t.tv_nsec*1e-6;}
typedef struct {double* dst; const uint8_t* idx; const double* dict; size_t n;} Job;
static void* expand(void* p){Job* j=p; for(size_t i=0;i<j->n;i++) j->dst[i]=j->dict[j->idx[i]]; return 0;}
int main(int argc,char**argv){
  size_t n=19333781; int T=argc>1?atoi(argv[1]):8;
  double* v=malloc(n*8); int32_t* a=malloc(n*4); uint8_t* idx=malloc(n); double dict[256];
  for(int i=0;i<256;i++) dict[i]=i*0.5; memset(idx,3,n); memset(v,0,n*8); memset(a,0,n*4);
  for(int rep=0;rep<3;rep++){
    double t0=now(); pthread_t th[64]; Job jb[64];
    for(int k=0;k<T;k++){jb[k].dst=v+n*k/T; jb[k].idx=idx+n*k/T; jb[k].dict=dict; jb[k].n=n*(k+1)/T-n*k/T; pthread_create(&th[k],0,expand,&jb[k]);}
    for(int k=0;k<T;k++) pthread_join(th[k],0);
    double t1=now();
    printf("T=%d expand 155MB: %.2f ms (%.1f GB/s)\n",T,t1-t0,n*9/1e6/(t1-t0));
  }
  return 0;
}
