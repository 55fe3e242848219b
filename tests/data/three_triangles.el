# three triangles sharing vertices 2 and 4
0 1
1 2
0 2
2 3
3 4
2 4
4 5
5 6
4 6
