# complete graph on 4 vertices
0 1
0 2
0 3
1 2
1 3
2 3
